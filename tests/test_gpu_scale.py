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
def test_parity_at_scale(N, d, kernel, variant, eps):
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
