"""The exporter on a live reference HierRep (runs where /root/reference is
present, i.e. the build container; skipped elsewhere): every store= choice of
export_rep -- the path GpuHierRep.from_rep(rep, recompute=...) takes -- gives
the reference's own matvec through the oracle, and not-stored blocks are
really absent from the blob."""

import os
import sys

import numpy as np
import pytest

from golden_io import rel_err
from oracle.packed_matvec import packed_matvec

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package absent")


@pytest.fixture(scope="module")
def ref_rep():
    sys.path.insert(0, REF)
    import h2weak as h
    pts = h.make_points("uniform", 600, 3, 42)
    tree = h.build_tree(pts, 12)
    rep = h.build_variant("h2plusH-star", tree, h.make_kernel("lap3d", pts), eps=1e-6)
    q = np.random.default_rng(43).standard_normal(600)
    return rep, q, rep.matvec(q)


@pytest.mark.parametrize("store", ["near,m2l", "near", "m2l", ""])
def test_export_store_choices(ref_rep, store):
    from paper_2309_14085_b200.export import export_rep
    rep, q, phi_ref = ref_rep
    op = export_rep(rep, store=store)
    assert (op.near_off >= 0).all() == ("near" in store)
    assert all((ch.m2l_off >= 0).all() == ("m2l" in store) for ch in op.channels)
    assert op.mem_scalars == rep.mem_scalars
    assert rel_err(packed_matvec(op, q), phi_ref) <= 1e-13
    full = export_rep(rep)
    if store != "near,m2l":
        assert len(op.blob) < len(full.blob)


def test_from_rep_needs_points_for_evaluation(ref_rep):
    from paper_2309_14085_b200.export import export_rep
    rep, q, phi_ref = ref_rep
    with pytest.raises(ValueError, match="with_points"):
        export_rep(rep, with_points=False, store="near")


def test_from_rep_is_loud_without_gpu(ref_rep):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    rep, q, phi_ref = ref_rep
    with pytest.raises(RuntimeError):
        GpuHierRep.from_rep(rep, recompute="m2l,near")
