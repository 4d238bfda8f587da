"""Pin the oracle (oracle/packed_matvec.py) against the reference's own
``HierRep.matvec`` outputs stored in the golden fixtures.  Tolerance 1e-13 (2-norm relative): the
only difference is fp64 summation order inside transposed BLAS GEMVs.

The fixtures were produced by tests/golden/make_golden.py from the reference
(engine.py:250-269 on the operator built by engine.py:325-373)."""

import numpy as np
import pytest

from golden_io import golden_names, load_golden, rel_err
from oracle.packed_matvec import dense_matvec_points, packed_matvec

NAMES = golden_names()


def test_fixtures_present():
    assert len(NAMES) >= 8


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_matvec(name):
    op, z, meta = load_golden(name)
    phi = packed_matvec(op, z["q"])
    assert rel_err(phi, z["phi_ref"]) <= 1e-13
    for j in range(z["Q"].shape[1]):
        assert rel_err(packed_matvec(op, z["Q"][:, j]), z["Phi_ref"][:, j]) <= 1e-13


@pytest.mark.parametrize("name", NAMES)
def test_oracle_dense_restatement(name):
    """The dense restatement of kernels.py:36-57 reproduces the reference's
    dense oracle (bench.py:87-97) and thus its own RE_MVP."""
    op, z, meta = load_golden(name)
    pts = np.empty_like(op.points_tree)
    pts[op.perm] = op.points_tree
    dense = dense_matvec_points(pts, op.kernel, z["q"])
    assert rel_err(dense, z["phi_dense"]) <= 1e-13
    assert abs(rel_err(z["phi_ref"], dense) - meta["re_ref"]) <= 1e-3 * meta["re_ref"] + 1e-15


@pytest.mark.parametrize("name", NAMES)
def test_export_tally(name):
    """Packed scalars equal the reference's mem_scalars tally
    (engine.py:184-186, 315; blr.py:59) for non-symmetric builds."""
    op, z, meta = load_golden(name)
    assert op.stored_scalars() == op.mem_scalars == meta["mem_scalars"]


def test_length_mismatch():
    op, z, _ = load_golden(NAMES[0])
    with pytest.raises(ValueError, match="vector length mismatch"):
        packed_matvec(op, np.zeros(op.N + 1))
