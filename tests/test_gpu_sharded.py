"""Sharded GPU plans on ONE device: R virtual ranks run their halves one
after the other (no kernel waits on another), the all-gather is emulated by
concatenating the packed buffers.  Exercises the real sharded plans
(h2g_plan_create_sharded, begin / pack / unpack / end) end to end."""

import numpy as np
import pytest

from golden_io import golden_names, load_golden, rel_err

pytestmark = pytest.mark.gpu


def _virtual_ranks(op, q, R):
    import torch
    from paper_2309_14085_b200.sharded import ShardedGpuHierRep
    reps = [ShardedGpuHierRep(op, r, R, device=0) for r in range(R)]
    qd = torch.from_numpy(np.asarray(q, dtype=np.float64)).cuda()
    stream = torch.cuda.current_stream().cuda_stream
    mx = max(1, reps[0].info["max_send_slots"])
    recv = torch.zeros(mx * R, dtype=torch.float64, device="cuda")
    for r, rep in enumerate(reps):
        send = torch.zeros(mx, dtype=torch.float64, device="cuda")
        rep.begin(qd, stream)
        rep.pack(send, stream)
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


@pytest.mark.parametrize("R", [2, 4])
@pytest.mark.parametrize("name", golden_names())
def test_virtual_ranks_match_reference(name, R):
    op, z, meta = load_golden(name)
    phi, infos = _virtual_ranks(op, z["q"], R)
    assert rel_err(phi, z["phi_ref"]) <= 1e-12
    assert sum(i["row_end"] - i["row_begin"] for i in infos) == op.N


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
