"""GPU parity at the BASELINE.json configuration sizes.

The reference's own Python build is infeasible at these sizes (~30 min at
N=1M), so the operator comes from the native builder, which reproduces the
reference's construction (tests/test_builder.py: identical trees, lists,
ranks; matvec equal to the reference's own to roundoff).  On that operator:

* north-star check 1: GPU matvec vs the oracle restatement of the
  reference's matvec (oracle/packed_matvec.py, pinned to the reference's
  golden outputs) -- relative 2-norm error <= 1e-12;
* north-star check 2: on a seeded sample of target rows, the error of the
  GPU result against the direct dense product equals the reference
  algorithm's own error (the oracle's) up to the 1e-12-level difference of
  the two results (absolute slack 1e-11 in relative-error units).
"""

import numpy as np
import pytest

from golden_io import rel_err
from oracle.packed_matvec import dense_matvec_points, packed_matvec
from paper_2309_14085_b200.builder import build_variant, uniform_points

pytestmark = pytest.mark.gpu

CASES = [
    # (N, d, kernel, variant, eps)   cfg1 / cfg2 of BASELINE.json + a 3D case
    (4096, 2, "log2d", "h2star-bt", 1e-8),
    (4096, 2, "log2d", "h2plusH-star", 1e-8),
    (1048576, 2, "log2d", "h2star-bt", 1e-8),
    (1048576, 2, "log2d", "h2plusH-star", 1e-8),
    (65536, 3, "lap3d", "h2star-bt", 1e-6),
    (65536, 3, "lap3d", "h2plusH-star", 1e-6),
]


@pytest.mark.parametrize("N,d,kernel,variant,eps", CASES)
def test_parity_at_scale(N, d, kernel, variant, eps, capsys):
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    pts = uniform_points(N, d, 42)
    op = build_variant(variant, pts, kernel, 64, eps)
    q = np.random.default_rng(43).standard_normal(N)
    with GpuHierRep(op) as rep:
        phi = rep.matvec(q)
        assert np.array_equal(phi, rep.matvec(q))  # bitwise repeatable
        # batched-RHS engine at scale (group mode on the wide phases): 16 RHS
        Q = np.random.default_rng(44).standard_normal((N, 16))
        Q[:, 3] = q
        Phi = rep.matmat(Q)
        assert rel_err(Phi[:, 11], rep.matvec(Q[:, 11])) <= 2e-12
    ref = packed_matvec(op, q)
    assert rel_err(phi, ref) <= 1e-12
    assert rel_err(Phi[:, 3], ref) <= 1e-12
    rows = np.sort(np.random.default_rng(7).choice(N, size=min(N, 128), replace=False))
    exact = dense_matvec_points(pts, op.kernel, q, block=8, rows=rows)
    re_gpu = rel_err(phi[rows], exact)
    re_ref = rel_err(ref[rows], exact)
    assert abs(re_gpu - re_ref) <= 1e-11
    if N == 1048576:  # parity margin vs a long-double evaluation (cfg 2)
        from oracle.packed_matvec import packed_matvec_rows
        lo = op.level_offset
        leaves = np.random.default_rng(5).choice(np.arange(lo[op.kappa], lo[op.kappa + 1]), 24,
                                                 replace=False)
        r_ld, v_ld = packed_matvec_rows(op, q, leaves, dtype=np.longdouble)
        v_ld = v_ld.astype(np.float64)
        m_gpu, m_orc = rel_err(phi[r_ld], v_ld), rel_err(ref[r_ld], v_ld)
        assert m_gpu <= 1e-12
        with capsys.disabled():
            print(f"\ncfg2 {variant} margin: gpu_vs_oracle={rel_err(phi, ref):.2e} "
                  f"gpu_vs_longdouble={m_gpu:.2e} oracle_vs_longdouble={m_orc:.2e}")
    if N <= 65536:
        # reference acceptance criterion 1 (test_acceptance.py:54-83, checked there
        # at N <= 5000).  At N = 1M the reference algorithm's own error grows past
        # it for H2*(b+t) (1.1e-5 at eps 1e-8, identical for oracle and GPU; the
        # native build equals the reference build, tests/test_builder.py).
        assert re_gpu <= 100 * eps


@pytest.mark.parametrize("variant", ["h2star-bt", "h2plusH-star"])
def test_tall_blocks_as_row_panels(variant):
    """Near blocks taller than 256 rows (leaves of up to 400 points) stream as
    row panels (contiguous pieces): single- and 16-RHS results equal the
    oracle on the export's own layout."""
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op = build_variant(variant, uniform_points(6000, 2, 42), "log2d", 400, 1e-8)
    q = np.random.default_rng(43).standard_normal(op.N)
    ref = packed_matvec(op, q)
    Q = np.random.default_rng(3).standard_normal((op.N, 16))
    with GpuHierRep(op) as rep:
        assert rel_err(rep.matvec(q), ref) <= 1e-12
        Phi = rep.matmat(Q)
    for j in (0, 9, 15):
        assert rel_err(Phi[:, j], packed_matvec(op, Q[:, j])) <= 1e-12


def _margins(phi_rows, oracle_rows, ld_rows):
    ld = ld_rows.astype(np.float64)
    return {"gpu_vs_oracle": rel_err(phi_rows, oracle_rows),
            "gpu_vs_longdouble": rel_err(phi_rows, ld),
            "oracle_vs_longdouble": rel_err(oracle_rows, ld)}


@pytest.fixture(scope="module")
def cfg3_op():
    """BASELINE configs[2] exactly: uniform_points(1048576, 3, 42), 1/r, leaf
    <= 64, eps 1e-6, H2*(b+t), every block stored (89.8 GB)."""
    from paper_2309_14085_b200.builder import build_variant, uniform_points
    pts = uniform_points(1 << 20, 3, 42)
    op = build_variant("h2star-bt", pts, "lap3d", 64, 1e-6)
    yield op, pts
    del op


def test_cfg3_streamed_vs_evaluated_vs_oracle(cfg3_op, capsys):
    """North-star HBM config (cfg 3) at full size, both operating modes:

    * streamed (every block read from HBM) vs M2L evaluated (the bench's
      headline mode, all evaluated and with the bench's staged share) vs
      near + M2L evaluated: each <= 1e-12 from the others over all N rows;
    * each vs the oracle restatement of the reference matvec on 48 sampled
      target leaves (packed_matvec_rows: full upward pass, the leaves'
      ancestor chains) <= 1e-12;
    * the parity margin: GPU and oracle against a long-double evaluation of
      the same operator on 12 of those leaves;
    * 128 sampled rows of the direct dense product: the GPU's error equals
      the reference algorithm's own (the oracle's)."""
    from oracle.packed_matvec import packed_matvec_rows
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op, pts = cfg3_op
    N = op.N
    q = np.random.default_rng(43).standard_normal(N)
    import bench
    res = {}
    # "m2l@staged": the bench's headline plan (a share of every target's M2L
    # blocks evaluated, the rest TMA-staged by the P2P CTAs' streaming warps)
    for key, mode, share in (("", "", 1.0), ("m2l", "m2l", 1.0),
                             ("m2l@staged", "m2l", bench.M2L_EVAL_SHARE),
                             ("near,m2l", "near,m2l", 1.0)):
        with GpuHierRep(op, recompute=mode, m2l_share=share) as rep:
            res[key] = rep.matvec(q)
            assert np.array_equal(res[key], rep.matvec(q))
    for key in ("m2l", "m2l@staged", "near,m2l"):
        assert rel_err(res[key], res[""]) <= 1e-12, key
    lo = op.level_offset
    rng = np.random.default_rng(11)
    leaves = rng.choice(np.arange(lo[op.kappa], lo[op.kappa + 1]), 48, replace=False)
    rows, orc = packed_matvec_rows(op, q, leaves)
    for mode, phi in res.items():
        assert rel_err(phi[rows], orc) <= 1e-12, mode
    rows_ld, ld = packed_matvec_rows(op, q, leaves[:12], dtype=np.longdouble)
    k = len(rows_ld)
    margins = {mode or "streamed": _margins(phi[rows_ld], orc[:k], ld) for mode, phi in res.items()}
    for m in margins.values():
        assert m["gpu_vs_longdouble"] <= 1e-12
    drows = np.sort(np.random.default_rng(7).choice(N, size=128, replace=False))
    exact = dense_matvec_points(pts, op.kernel, q, block=8, rows=drows)
    mask = np.isin(drows, rows)
    re_gpu = rel_err(res["m2l"][drows], exact)
    # oracle at the dense rows: the rows' own leaves
    tree_pos = np.empty(N, dtype=np.int64)
    tree_pos[op.perm] = np.arange(N)
    dleaves = np.unique(np.searchsorted(op.cl_start[lo[op.kappa]:lo[op.kappa + 1]],
                                        tree_pos[drows], side="right") - 1 + lo[op.kappa])
    r2, o2 = packed_matvec_rows(op, q, dleaves)
    orc_d = dict(zip(r2.tolist(), o2.tolist()))
    re_orc = rel_err(np.array([orc_d[i] for i in drows]), exact)
    assert abs(re_gpu - re_orc) <= 1e-11
    with capsys.disabled():
        print(f"\ncfg3 parity: N={N} kappa={op.kappa} mem_scalars={op.mem_scalars} "
              f"dense-sample error gpu={re_gpu:.3e} oracle={re_orc:.3e} (rows sampled {mask.sum()})")
        for mode, m in margins.items():
            print(f"cfg3 margin [{mode}]: " + " ".join(f"{a}={b:.2e}" for a, b in m.items()))
