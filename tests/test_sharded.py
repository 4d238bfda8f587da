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
from oracle.sched_emulator import emulate_begin, emulate_end, emulate_matvec
from paper_2309_14085_b200.sharded import schedule_view

NAMES = golden_names()
SMALL = NAMES


@pytest.mark.parametrize("name", NAMES)
def test_single_rank_schedule_is_the_reference_matvec(name):
    op, z, meta = load_golden(name)
    assert rel_err(emulate_matvec(op, z["q"], 1), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
@pytest.mark.parametrize("name", SMALL)
def test_sharded_schedules_compose(name, nranks):
    op, z, meta = load_golden(name)
    assert rel_err(emulate_matvec(op, z["q"], nranks), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["g2d_log_h2plusH", "g3d_lap_h2star", "g3d_lap_h2plusH",
                                  "g3d_lap_k3_h2star", "g3d_gauss_k3_h2star"])
def test_sharded_evaluated_blocks(name, nranks):
    """Config 5's operating mode: near and M2L blocks NOT stored (evaluated
    from the points / NCA pivots on every rank) and subtree-sharded.  The
    evaluated terms of every rank's schedule reproduce the reference's
    matvec on its stored operator (engine.py:176-179, 309-318)."""
    op, z, meta = load_golden(name)
    ev = op.without_blocks(near=True, m2l=True)
    assert rel_err(emulate_matvec(ev, z["q"], nranks), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("recompute", ["near", "m2l", "near,m2l"])
def test_sharded_recompute_mask_on_stored_operator(recompute):
    """Blocks evaluated although stored (the recompute mask), sharded x 4."""
    op, z, meta = load_golden("g3d_lap_h2star")
    v = schedule_view(op, 1, 4, recompute)
    assert (v["terms"][:, 4] == 2).any()
    assert rel_err(emulate_matvec(op, z["q"], 4, recompute), z["phi_ref"]) <= 1e-13


def _worker(rank, world, port, name, out_path, unstored=False):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    import torch
    from golden_io import load_golden
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    op, z, meta = load_golden(name)
    if unstored:
        op = op.without_blocks(near=True, m2l=True)
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


@pytest.mark.parametrize("name,unstored", [("g2d_log_h2plusH", False), ("g3d_lap_h2star", False),
                                           ("g3d_lap_h2plusH", True), ("g3d_lap_k3_h2star", True)])
def test_gloo_world_size_2(tmp_path, name, unstored):
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = str(tmp_path / "phi.npy")
    mp.spawn(_worker, args=(2, port, name, out, unstored), nprocs=2, join=True)
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
    # row panels applied in place; (H2+H)*: stacked BLR V^T factors appended
    assert len(view["blob"]) >= len(op.blob)
    assert (len(view["blob"]) > len(op.blob) + 1) == (variant == "h2plusH-star")
    assert not np.array_equal(view["blob"][:len(op.blob)], op.blob)
    assert rel_err(emulate_matvec(op, q, 1), ref) <= 1e-13
    assert rel_err(emulate_matvec(op, q, 2), ref) <= 1e-13


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("name,unstored", [("g2d_log_h2plusH", False), ("g3d_lap_h2plusH", True),
                                           ("g3d_lap_k3_h2star", True), ("g2d_cfg1_h2plusH", True)])
def test_distributed_q_with_x_halo(name, unstored, nranks):
    """Distributed vectors: every rank starts with ONLY its own rows of q
    (the others NaN); the x-halo all-gather (near sources, BLR V^T sources
    across subtree boundaries) supplies exactly what its schedule reads, and
    the result is the reference's matvec."""
    from oracle.sched_emulator import emulate_matvec_distributed
    op, z, meta = load_golden(name)
    if unstored:
        op = op.without_blocks(near=True, m2l=True)
    phi = emulate_matvec_distributed(op, z["q"], nranks)
    assert np.isfinite(phi).all()
    assert rel_err(phi, z["phi_ref"]) <= 1e-13
    v = schedule_view(op, 0, nranks)
    halo_rows = int(v["halo"][:, 2].sum())
    assert halo_rows < op.N  # a halo, not a replicated q


def test_shard_level_follows_north_star():
    """Subtrees at level 3 when the tree is that deep."""
    op, z, meta = load_golden("g3d_lap_k3_h2star")
    for R in (2, 4, 8):
        assert schedule_view(op, 0, R)["level"] == 3


def test_blr_factors_stacked_by_source(monkeypatch):
    """Unsharded (H2+H)* schedules apply the BLR stage-1 factors V_XY^T that
    share a source Y as ONE task (rows concatenated in an extension of the
    blob, one x segment q_Y; w = V^T q_Y, blr.py:83): fewer, larger stage-1
    tasks, same result as the reference's matvec either way."""
    op, z, meta = load_golden("g2d_cfg1_h2plusH")
    stacked = schedule_view(op, 0, 1)
    phi = emulate_matvec(op, z["q"], 1)
    monkeypatch.setenv("H2G_BLR_STACK", "0")
    plain = schedule_view(op, 0, 1)
    phi0 = emulate_matvec(op, z["q"], 1)
    n_vq = lambda v: int(v["phases"][1][1] - v["phases"][1][0])   # phase 1 = blr_vq
    assert n_vq(stacked) < n_vq(plain)
    assert len(stacked["blob"]) > len(op.blob) and len(plain["blob"]) == 0
    assert int(stacked["tasks"][stacked["phases"][1][0]:stacked["phases"][1][1], 1].max()) <= 256
    assert rel_err(phi, z["phi_ref"]) <= 1e-13 and rel_err(phi0, z["phi_ref"]) <= 1e-13
