"""Sharded GPU plans on ONE device: R virtual ranks run their halves one
after the other (no kernel waits on another), the all-gathers are emulated by
concatenating the packed buffers.  Exercises the real sharded plans
(h2g_plan_create_sharded, begin / pack / unpack / end, and the distributed
vector path with its x-halo exchange) end to end, including config 5's
operating mode: near and M2L blocks not stored, evaluated on every rank."""

import numpy as np
import pytest

from golden_io import golden_names, load_golden, rel_err

pytestmark = pytest.mark.gpu


def _virtual_ranks(op, q, R, recompute="", m2l_share=1.0):
    import torch
    from paper_2309_14085_b200.sharded import ShardedGpuHierRep
    reps = [ShardedGpuHierRep(op, r, R, device=0, recompute=recompute, m2l_share=m2l_share)
            for r in range(R)]
    qd = torch.from_numpy(np.asarray(q, dtype=np.float64)).cuda()
    stream = torch.cuda.current_stream().cuda_stream
    mx = max(1, reps[0].info["max_send_slots"])
    recv = torch.zeros(mx * R, dtype=torch.float64, device="cuda")
    for r, rep in enumerate(reps):
        send = torch.zeros(mx, dtype=torch.float64, device="cuda")
        rep.begin(qd, stream)
        rep.pack(send, stream)
        if r % 2 == 0:  # the owned near field beside the exchange, as matvec() does;
            rep.overlap(stream)  # odd ranks leave it to end()
        recv[r * mx:(r + 1) * mx] = send
    phi = torch.zeros_like(qd)
    for rep in reps:
        part = torch.zeros_like(qd)
        rep.unpack(recv, stream)
        rep.end(part, stream)
        phi += part
    torch.cuda.synchronize()
    infos = [rep.info for rep in reps]
    for rep in reps:
        rep.close()
    return phi.cpu().numpy(), infos


def _virtual_ranks_distributed(op, q, R, recompute=""):
    """Distributed vectors: rank r holds only q[perm[row_begin:row_end]]."""
    import ctypes as C
    import torch
    from paper_2309_14085_b200 import _lib
    from paper_2309_14085_b200.sharded import ShardedGpuHierRep
    reps = [ShardedGpuHierRep(op, r, R, device=0, recompute=recompute) for r in range(R)]
    stream = torch.cuda.current_stream().cuda_stream
    s = C.c_void_p(stream)
    q_tree = torch.from_numpy(np.asarray(q, dtype=np.float64)[op.perm]).cuda()
    hm = max(1, reps[0].info["max_halo_slots"])
    mx = max(1, reps[0].info["max_send_slots"])
    hrecv = torch.zeros(hm * R, dtype=torch.float64, device="cuda")
    recv = torch.zeros(mx * R, dtype=torch.float64, device="cuda")
    for r, rep in enumerate(reps):
        rb, re_ = rep.owned_rows()
        q_own = q_tree[rb:re_].clone()
        _lib.check(rep._L.h2g_shard_load_q(rep._plan, C.c_void_p(q_own.data_ptr()), s))
        hsend = torch.zeros(hm, dtype=torch.float64, device="cuda")
        _lib.check(rep._L.h2g_halo_pack(rep._plan, C.c_void_p(hsend.data_ptr()), s))
        hrecv[r * hm:(r + 1) * hm] = hsend
    for r, rep in enumerate(reps):
        _lib.check(rep._L.h2g_halo_unpack(rep._plan, C.c_void_p(hrecv.data_ptr()), s))
        _lib.check(rep._L.h2g_shard_part0(rep._plan, s))
        send = torch.zeros(mx, dtype=torch.float64, device="cuda")
        rep.pack(send, stream)
        recv[r * mx:(r + 1) * mx] = send
    phi_tree = torch.full_like(q_tree, float("nan"))
    for rep in reps:
        rb, re_ = rep.owned_rows()
        rep.unpack(recv, stream)
        out = torch.empty(re_ - rb, dtype=torch.float64, device="cuda")
        _lib.check(rep._L.h2g_shard_store_phi(rep._plan, C.c_void_p(out.data_ptr()), s))
        phi_tree[rb:re_] = out
    torch.cuda.synchronize()
    for rep in reps:
        rep.close()
    phi = np.empty(op.N)
    phi[op.perm] = phi_tree.cpu().numpy()
    return phi


@pytest.mark.parametrize("R", [2, 4])
@pytest.mark.parametrize("name", golden_names())
def test_virtual_ranks_match_reference(name, R):
    op, z, meta = load_golden(name)
    phi, infos = _virtual_ranks(op, z["q"], R)
    assert rel_err(phi, z["phi_ref"]) <= 1e-12
    assert sum(i["row_end"] - i["row_begin"] for i in infos) == op.N


@pytest.mark.parametrize("R", [2, 8])
@pytest.mark.parametrize("name", ["g2d_log_h2plusH", "g3d_lap_h2star", "g3d_lap_h2plusH",
                                  "g3d_lap_k3_h2star", "g3d_lap_k3_h2plusH",
                                  "g3d_gauss_k3_h2star"])
def test_virtual_ranks_evaluated_blocks(name, R):
    """Config 5's mode: no near / M2L block stored, all evaluated on the P2P
    engine of every rank; equals the reference's matvec."""
    op, z, meta = load_golden(name)
    ev = op.without_blocks(near=True, m2l=True)
    phi, infos = _virtual_ranks(ev, z["q"], R)
    assert rel_err(phi, z["phi_ref"]) <= 1e-12


@pytest.mark.parametrize("recompute", ["m2l", "near,m2l"])
def test_virtual_ranks_recompute_mask(recompute):
    op, z, meta = load_golden("g3d_lap_h2plusH")
    phi, infos = _virtual_ranks(op, z["q"], 4, recompute=recompute)
    assert rel_err(phi, z["phi_ref"]) <= 1e-12


@pytest.mark.parametrize("name", ["g3d_lap_k3_h2star", "g3d_lap_k3_h2plusH"])
def test_virtual_ranks_staged_share(name):
    """The bench's multi-GPU mode: every rank evaluates a share of its M2L
    entries and stages the rest through its P2P CTAs' streaming warps."""
    op, z, meta = load_golden(name)
    phi, infos = _virtual_ranks(op, z["q"], 4, recompute="m2l", m2l_share=0.6)
    assert rel_err(phi, z["phi_ref"]) <= 1e-12


@pytest.mark.parametrize("R", [2, 8])
@pytest.mark.parametrize("name,unstored", [("g2d_log_h2plusH", False), ("g3d_lap_k3_h2plusH", True),
                                           ("g2d_cfg1_h2star", True)])
def test_virtual_ranks_distributed_vectors(name, unstored, R):
    """q and phi distributed by owned tree rows; x halo exchanged."""
    op, z, meta = load_golden(name)
    if unstored:
        op = op.without_blocks(near=True, m2l=True)
    phi = _virtual_ranks_distributed(op, z["q"], R)
    assert np.isfinite(phi).all()
    assert rel_err(phi, z["phi_ref"]) <= 1e-12


def test_virtual_ranks_at_scale():
    """cfg 2 (2D N=1M) split over 4 ranks equals the single-GPU plan; every
    rank holds a fraction of the operator."""
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op = build_variant("h2star-bt", uniform_points(1 << 20, 2, 42), "log2d", 64, 1e-8)
    q = np.random.default_rng(43).standard_normal(op.N)
    with GpuHierRep(op) as rep:
        ref = rep.matvec(q)
    phi, infos = _virtual_ranks(op, q, 4)
    assert rel_err(phi, ref) <= 1e-12
    assert max(i["blob_bytes"] for i in infos) < 0.35 * 8 * len(op.blob)


def test_virtual_ranks_cfg5_mode_at_scale():
    """Config 5's generator and mode at 1/64 of its size: jittered 64^3 grid,
    1/r, leaf <= 64, eps 1e-6, only the transfer operators stored; subtrees
    at level 3 over 8 ranks vs the 1-GPU plan, and the distributed-vector
    path (x halo) vs the same."""
    from paper_2309_14085_b200.builder import build_variant, jittered_grid
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op = build_variant("h2star-bt", jittered_grid(64, 3, 42), "lap3d", 64, 1e-6, store="")
    q = np.random.default_rng(43).standard_normal(op.N)
    with GpuHierRep(op) as rep:
        ref = rep.matvec(q)
    phi, infos = _virtual_ranks(op, q, 8)
    assert all(i["level"] == 3 for i in infos)
    assert rel_err(phi, ref) <= 1e-12
    phi_d = _virtual_ranks_distributed(op, q, 8)
    assert rel_err(phi_d, ref) <= 1e-12
