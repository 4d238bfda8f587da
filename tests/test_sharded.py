"""Multi-GPU sharding logic on CPU.

The per-rank schedules come from the same C++ code the GPU plans use
(h2g_schedule_build, include/h2g.h); a numpy emulator executes them.  The
sharded result must equal the reference's own matvec (golden fixtures) for
every rank count, with the exchange done by gloo all-gather across processes.
"""

import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import golden_names, load_golden, rel_err
from paper_2309_14085_b200.sharded import (emulate_begin, emulate_end, emulate_matvec,
                                           schedule_view)

NAMES = golden_names()


@pytest.mark.parametrize("name", NAMES)
def test_single_rank_schedule_is_the_reference_matvec(name):
    op, z, meta = load_golden(name)
    assert rel_err(emulate_matvec(op, z["q"], 1), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
@pytest.mark.parametrize("name", NAMES)
def test_sharded_schedules_compose(name, nranks):
    op, z, meta = load_golden(name)
    assert rel_err(emulate_matvec(op, z["q"], nranks), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("name", ["g2d_log_h2plusH", "g3d_lap_h2star"])
def test_rows_partition_and_blob_compaction(name):
    op, z, meta = load_golden(name)
    R = 4
    views = [schedule_view(op, r, R) for r in range(R)]
    bounds = [(v["row_begin"], v["row_end"]) for v in views]
    assert bounds[0][0] == 0 and bounds[-1][1] == op.N
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(R - 1))
    sizes = [len(v["blob"]) for v in views]
    assert max(sizes) < len(op.blob)            # each rank holds a fraction
    assert sum(sizes) < 1.5 * len(op.blob)      # replication limited to coarse levels
    assert all(v["max_send_slots"] == views[0]["max_send_slots"] for v in views)


def _worker(rank, world, port, name, out_path):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    import torch
    from golden_io import load_golden
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    op, z, meta = load_golden(name)
    v = schedule_view(op, rank, world)
    arena, send = emulate_begin(v, op, z["q"])
    send_t = torch.from_numpy(send[:max(1, v["max_send_slots"])].copy())
    recv_t = torch.zeros(send_t.numel() * world, dtype=torch.float64)
    dist.all_gather_into_tensor(recv_t, send_t)
    phi = torch.from_numpy(emulate_end(v, op, arena, recv_t.numpy()))
    dist.all_reduce(phi)  # disjoint rows
    if rank == 0:
        np.save(out_path, phi.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["g2d_log_h2plusH", "g3d_lap_h2star"])
def test_gloo_world_size_2(tmp_path, name):
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = str(tmp_path / "phi.npy")
    mp.spawn(_worker, args=(2, port, name, out), nprocs=2, join=True)
    op, z, meta = load_golden(name)
    assert rel_err(np.load(out), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("nranks", [1, 3])
@pytest.mark.parametrize("name", ["g2d_log_bigleaf_h2star", "g2d_log_h2plusH", "g3d_lap_h2star"])
def test_split_k_heavy_tasks(monkeypatch, name, nranks):
    """Heavy tasks cut into split-K pieces + reduce phases (forced here by a
    tiny piece floor) still compose to the reference matvec."""
    op, z, meta = load_golden(name)
    plain = schedule_view(op, 0, nranks)["phases"]
    monkeypatch.setenv("H2G_SPLIT_MIN_BYTES", "2048")
    v = schedule_view(op, 0, nranks)
    # reduce phases carry no algorithmic bytes
    n_red = int((v["phases"][:, 3] == 0).sum()) - int((plain[:, 3] == 0).sum())
    assert n_red >= 1 and len(v["phases"]) == len(plain) + n_red
    assert rel_err(emulate_matvec(op, z["q"], nranks), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("variant", ["h2star-bt", "h2plusH-star"])
def test_tall_blocks_as_row_panels(variant):
    """Leaves of up to 400 points make near blocks taller than the 256-row task
    limit: the unsharded schedule applies them as row pieces of blocks moved
    to row-panel layout (panelize_tall_blocks); the schedule over that blob
    equals the oracle, and a sharded schedule (no panels) too."""
    from oracle.packed_matvec import packed_matvec
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    op = build_variant(variant, uniform_points(6000, 2, 42), "log2d", 400, 1e-8)
    q = np.random.default_rng(43).standard_normal(op.N)
    ref = packed_matvec(op, q)
    view = schedule_view(op, 0, 1)
    assert len(view["blob"]) == len(op.blob)            # row panels applied
    assert not np.array_equal(view["blob"], op.blob)
    assert rel_err(emulate_matvec(op, q, 1), ref) <= 1e-13
    assert rel_err(emulate_matvec(op, q, 2), ref) <= 1e-13
