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
    assert len(NAMES) >= 13
    # BASELINE configs[0] exactly, both variants, and 3D trees of depth >= 3
    for name in ("g2d_cfg1_h2star", "g2d_cfg1_h2plusH", "g3d_lap_k3_h2star",
                 "g3d_lap_k3_h2plusH", "g3d_gauss_k3_h2star"):
        op, z, meta = load_golden(name)
        assert meta["kappa"] >= 3 and meta["N"] == 4096


def test_cfg1_fixture_is_baseline_config0():
    """configs[0]: uniform_points(4096, 2, 42), log r, leaf <= 64, eps 1e-8."""
    from paper_2309_14085_b200.builder import uniform_points
    for name in ("g2d_cfg1_h2star", "g2d_cfg1_h2plusH"):
        op, z, meta = load_golden(name)
        assert (meta["dist"], meta["N"], meta["d"], meta["kernel"], meta["n_max"],
                meta["eps"], meta["seed"]) == ("uniform", 4096, 2, "log2d", 64, 1e-8, 42)
        pts = np.empty_like(op.points_tree)
        pts[op.perm] = op.points_tree
        assert np.array_equal(pts, uniform_points(4096, 2, 42))
        assert np.array_equal(z["q"], np.random.default_rng(43).standard_normal(4096))


@pytest.mark.parametrize("name", [n for n in NAMES if "k3" in n or "cfg1" in n])
def test_materialized_compact_fixture(name):
    """The compact fixtures' re-evaluated blocks give the reference's matvec
    through the stored-block path too."""
    from golden_io import materialize
    op, z, meta = load_golden(name)
    full = materialize(op)
    assert (full.near_off >= 0).all() and all((c.m2l_off >= 0).all() for c in full.channels)
    assert rel_err(packed_matvec(full, z["q"]), z["phi_ref"]) <= 1e-13


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


@pytest.mark.parametrize("name", NAMES)
def test_oracle_evaluated_blocks_match_reference(name):
    """Blocks marked "not stored" (offset -1) are evaluated from the points /
    NCA pivots by the oracle's restatement of Kernel.block (kernels.py:36-57):
    the result still matches the reference's matvec on its stored operator
    (engine.py:176-179: M2L = K[t_i, s_o]; engine.py:260-268 lazy near)."""
    op, z, meta = load_golden(name)
    assert all(ch.has_pivots for ch in op.channels)
    ev = op.without_blocks(near=True, m2l=True)
    ev.validate()
    assert rel_err(packed_matvec(ev, z["q"]), z["phi_ref"]) <= 1e-13


@pytest.mark.parametrize("name", NAMES)
def test_exported_pivots_reproduce_stored_m2l(name):
    """The exported pivots are the reference's: K[t_i(X), s_o(Y)] evaluated
    from them equals every stored M2L block (engine.py:176-179).  Compact
    fixtures hold no M2L blocks; make_golden.py measured the same difference
    against the reference's in-memory blocks when it wrote them (meta)."""
    from oracle.packed_matvec import kernel_block
    op, z, meta = load_golden(name)
    if meta.get("compact"):
        assert meta["blk_maxdiff_m2l"] <= 1e-15 and meta["blk_maxdiff_near"] <= 1e-15
        return
    worst = 0.0
    for ch in op.channels:
        for X in range(op.n_clusters):
            for k in range(ch.m2l_rowptr[X], ch.m2l_rowptr[X + 1]):
                Y = ch.m2l_src[k]
                M = op.mat(ch.m2l_off[k], ch.r_in[X], ch.r_out[Y])
                K = kernel_block(op, ch.piv_in[ch.piv_in_ptr[X]:ch.piv_in_ptr[X + 1]],
                                 ch.piv_out[ch.piv_out_ptr[Y]:ch.piv_out_ptr[Y + 1]])
                worst = max(worst, float(np.max(np.abs(M - K), initial=0.0)))
    assert worst <= 1e-15


@pytest.mark.parametrize("name", ["g2d_log_h2star", "g2d_log_h2plusH", "g3d_lap_k3_h2plusH",
                                  "g2d_cfg1_h2star", "g3d_gauss_k3_h2star"])
def test_restricted_oracle_equals_full(name):
    """packed_matvec_rows (the BASELINE-scale oracle on sampled target leaves)
    reproduces the full restatement's rows and the reference's own phi."""
    from oracle.packed_matvec import packed_matvec_rows
    op, z, meta = load_golden(name)
    lo = op.level_offset
    leaves = np.random.default_rng(1).choice(np.arange(lo[op.kappa], lo[op.kappa + 1]), 7,
                                             replace=False)
    rows, vals = packed_matvec_rows(op, z["q"], leaves)
    full = packed_matvec(op, z["q"])
    assert len(rows) == sum(op.size(x) for x in leaves)
    assert np.max(np.abs(vals - full[rows])) <= 1e-14 * np.max(np.abs(full))
    assert rel_err(vals, z["phi_ref"][rows]) <= 1e-13
    rows_ld, vals_ld = packed_matvec_rows(op, z["q"], leaves, dtype=np.longdouble)
    assert np.array_equal(rows_ld, rows)
    assert rel_err(vals, vals_ld.astype(np.float64)) <= 1e-13


def test_sampled_cpu_reference_timer():
    """bench.py's CPU reference leg: upward pass + one subtree's downward pass;
    the sampled rows it computes are the full restatement's."""
    from oracle.cpu_reference import sample_leaves, time_sampled_matvec
    from oracle.packed_matvec import downward_rows, upward_pass
    op, z, meta = load_golden("g3d_lap_k3_h2star")  # compact: blocks evaluated untimed
    leaves, L = sample_leaves(op, frac_level=2)
    assert L == 2 and len(leaves) == 8
    assert len(sample_leaves(op)[0]) == 512  # small tree: the whole matvec
    r = time_sampled_matvec(op, z["q"], steps=1)
    assert r["value"] > 0 and r["sampled_leaves"] == 512
    q_tree = z["q"][op.perm]
    out = downward_rows(op, q_tree, upward_pass(op, q_tree), leaves)
    full = packed_matvec(op, z["q"])
    for x in leaves:
        rows = op.perm[op.cl_start[x]:op.cl_end[x]]
        assert np.allclose(out[x], full[rows], rtol=0, atol=1e-13 * np.abs(full).max())
