"""GPU parity of the kernel-evaluation (P2P) engine, csrc/h2g_p2p.cuh.

The M2L blocks are raw kernel blocks K[t_i(X), s_o(Y)] (reference
engine.py:176-179) and the near blocks K[t^X, t^Y] (engine.py:309-318, lazily
evaluated by the reference itself with store_near=False), so the device may
evaluate them from the points / NCA pivots instead of streaming them.  Every
mode must still match the reference's own matvec on its stored operator to
the north-star tolerance (relative 2-norm <= 1e-12) and stay bitwise
repeatable; kernel entries follow Kernel.block (kernels.py:36-57), including
the r == 0 / i == j rules (Gaussian: zero_value 1 plus the diagonal shift).
"""

import numpy as np
import pytest

from golden_io import golden_names, load_golden, rel_err
from oracle.packed_matvec import packed_matvec

pytestmark = pytest.mark.gpu
NAMES = golden_names()
TOL = 1e-12
MODES = [("near", 1.0), ("m2l", 1.0), ("near,m2l", 1.0), ("near,m2l", 0.5), ("m2l", 0.6)]


@pytest.mark.parametrize("mode,share", MODES)
@pytest.mark.parametrize("name", NAMES)
def test_evaluated_blocks_match_reference(name, mode, share):
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op, z, meta = load_golden(name)
    with GpuHierRep(op, recompute=mode, m2l_share=share) as rep:
        st = rep.stats()
        phi = rep.matvec(z["q"])
        assert rel_err(phi, z["phi_ref"]) <= TOL
        assert np.array_equal(phi, rep.matvec(z["q"]))  # deterministic (no data atomics)
        assert st["n_launches"] >= 3
        Phi = rep.matmat(z["Q"])  # nrhs > 1: column loop through the same plan
        for j in range(z["Q"].shape[1]):
            assert rel_err(Phi[:, j], z["Phi_ref"][:, j]) <= TOL
        assert np.all(rep.matvec(np.zeros(op.N)) == 0)


@pytest.mark.parametrize("name", NAMES)
def test_unstored_blocks(name):
    """An export whose near and M2L blocks are not stored (offset -1) runs
    through the evaluation engine and matches the reference."""
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op, z, meta = load_golden(name)
    ev = op.without_blocks(near=True, m2l=True)
    with GpuHierRep(ev) as rep:
        assert rel_err(rep.matvec(z["q"]), z["phi_ref"]) <= TOL
        assert rel_err(rep.matvec(z["q"]), packed_matvec(ev, z["q"])) <= TOL


def test_coincident_points_use_zero_value():
    """Duplicate points (r == 0 off the diagonal) take zero_value; the
    diagonal takes (diag or zero_value) + shift -- kernels.py:41-55."""
    from paper_2309_14085_b200.builder import build_variant
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, (1500, 3))
    pts[700:760] = pts[100:160]  # coincident pairs in different leaves
    for kernel in ("lap3d", "gaussian"):
        op = build_variant("h2star-bt", pts, kernel, 24, 1e-6)
        q = rng.standard_normal(len(pts))
        ref = packed_matvec(op, q)
        with GpuHierRep(op.without_blocks(), device=0) as rep:
            assert rel_err(rep.matvec(q), ref) <= TOL


@pytest.mark.parametrize("N,d,kernel", [(2000, 2, "log2d"), (3000, 3, "lap3d")])
def test_big_leaves_row_split(N, d, kernel):
    """Leaves of ~500-750 points: near tasks are cut into <= 256-row pieces,
    including the self blocks whose i == j test must follow the row offset."""
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    pts = uniform_points(N, d, 9)
    op = build_variant("h2star-bt", pts, kernel, 600 if d == 2 else 500, 1e-10)
    assert int((op.cl_end - op.cl_start).max()) > 256
    q = np.random.default_rng(1).standard_normal(len(pts))
    ref = packed_matvec(op, q)
    for mode in ("near", "near,m2l"):
        with GpuHierRep(op, recompute=mode) as rep:
            assert rel_err(rep.matvec(q), ref) <= TOL


@pytest.mark.parametrize("N,d,kernel,eps", [(65536, 3, "lap3d", 1e-6),
                                            (262144, 2, "log2d", 1e-8)])
def test_at_scale_against_stored(N, d, kernel, eps):
    """At a large size: evaluated (both kinds, and the hybrid split) vs the
    streamed operator on the same build, and vs the oracle on a sample."""
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    pts = uniform_points(N, d, 42)
    op = build_variant("h2star-bt", pts, kernel, 64, eps)
    q = np.random.default_rng(43).standard_normal(N)
    with GpuHierRep(op) as rep:
        phi0 = rep.matvec(q)
    ref = packed_matvec(op, q)
    assert rel_err(phi0, ref) <= TOL
    for mode, share in (("near,m2l", 1.0), ("near,m2l", 0.6)):
        with GpuHierRep(op, recompute=mode, m2l_share=share) as rep:
            phi = rep.matvec(q)
            assert np.array_equal(phi, rep.matvec(q))
        assert rel_err(phi, ref) <= TOL


@pytest.mark.parametrize("nrhs", [16, 21])
@pytest.mark.parametrize("name", ["g2d_log_h2plusH", "g2d_cfg1_h2star", "g3d_lap_k3_h2star",
                                  "g3d_lap_k3_h2plusH", "g3d_gauss_k3_h2star"])
def test_batched_evaluated_engine(name, nrhs):
    """nrhs > 1 on plans with evaluated blocks: every kernel entry is evaluated
    once for all right-hand sides (csrc/h2g_p2p_batched.cuh) beside the
    tensor-pipe engine's stored blocks; equals the reference's matvec column
    by column (engine.py:250-269 applied to each column), bitwise repeatable,
    and the column loop (H2G_BATCHED_EVAL=0) to rounding."""
    import os
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op, z, meta = load_golden(name)
    reps = (nrhs + z["Q"].shape[1] - 1) // z["Q"].shape[1]
    Q = np.ascontiguousarray(np.tile(z["Q"], (1, reps))[:, :nrhs])
    Q[:, 1::2] *= -0.5  # distinct columns
    ref = np.tile(z["Phi_ref"], (1, reps))[:, :nrhs].copy()
    ref[:, 1::2] *= -0.5
    for mode, share, ev in (("m2l", 1.0, op), ("near,m2l", 0.6, op),
                            ("", 1.0, op.without_blocks(near=True, m2l=True))):
        with GpuHierRep(ev, recompute=mode, m2l_share=share) as rep:
            assert rep.launches_per_matvec(nrhs) < nrhs * rep.launches_per_matvec() // 2
            P = rep.matmat(Q)
            assert np.array_equal(P, rep.matmat(Q))
        for j in range(nrhs):
            assert rel_err(P[:, j], ref[:, j]) <= TOL, (mode, j)
    os.environ["H2G_BATCHED_EVAL"] = "0"
    try:
        with GpuHierRep(op, recompute="near,m2l") as rep:
            P0 = rep.matmat(Q)
    finally:
        os.environ.pop("H2G_BATCHED_EVAL")
    assert rel_err(P, P0) <= TOL
