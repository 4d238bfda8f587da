"""CPU-side checks of the C-ABI boundary: the library builds/loads, exports
every symbol include/h2g.h declares, and fails loudly without a GPU."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2309_14085_b200 import _lib
from paper_2309_14085_b200.build import build

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(h2g_[a-z0-9_]+)\s*\(", src)))


def test_build_and_load():
    build(verbose=False)
    L = _lib.load()
    assert L.h2g_abi_version() == _lib.H2G_ABI_VERSION


def test_every_declared_symbol_is_exported():
    L = _lib.load()
    declared = _declared("h2g.h")
    assert set(declared) == set(_lib.H2G_SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name


def test_error_strings():
    L = _lib.load()
    assert L.h2g_error_string(1) == b"vector length mismatch"
    assert L.h2g_error_string(0) == b"ok"


def test_bad_descriptor_rejected_without_gpu():
    L = _lib.load()
    d = _lib.ExportDesc()
    d.abi_version = 999
    plan = C.c_void_p()
    rc = L.h2g_plan_create(C.byref(d), 0, C.byref(plan))
    assert rc == 2 and not plan.value
    with pytest.raises(RuntimeError, match="bad export"):
        _lib.check(rc)


def _c_layout(struct, fields):
    """sizeof / offsetof of a struct in include/h2g.h, from the C compiler."""
    import subprocess
    import tempfile
    hdr = os.path.join(ROOT, "include", "h2g.h")
    body = "".join(f'printf("%zu\\n", offsetof({struct}, {f}));' for f in fields)
    src = (f'#include <stdio.h>\n#include <stddef.h>\n#include "{hdr}"\n'
           f'int main(void) {{ printf("%zu\\n", sizeof({struct})); {body} return 0; }}\n')
    with tempfile.TemporaryDirectory() as td:
        c = os.path.join(td, "layout.c")
        exe = os.path.join(td, "layout")
        with open(c, "w") as fh:
            fh.write(src)
        subprocess.run(["gcc", "-o", exe, c], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()
    return [int(x) for x in out]


@pytest.mark.parametrize("ctype,cname", [("ChannelDesc", "h2g_channel_desc"),
                                         ("ExportDesc", "h2g_export_desc"),
                                         ("PlanStats", "h2g_plan_stats"),
                                         ("ShardInfo", "h2g_shard_info")])
def test_struct_layout_matches_header(ctype, cname):
    """The ctypes mirrors in _lib.py have the C compiler's layout of h2g.h."""
    cls = getattr(_lib, ctype)
    names = [f for f, _ in cls._fields_]
    want = _c_layout(cname, names)
    got = [C.sizeof(cls)] + [getattr(cls, f).offset for f in names]
    assert got == want


def test_length_mismatch_maps_to_value_error():
    with pytest.raises(ValueError, match="vector length mismatch"):
        _lib.check(_lib.H2G_ERR_LENGTH_MISMATCH)


def test_no_device_is_loud():
    """Without a GPU the product path raises instead of falling back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from golden_io import golden_names, load_golden
    from paper_2309_14085_b200.gpu_rep import GpuHierRep
    op, _, _ = load_golden(golden_names()[0])
    with pytest.raises(RuntimeError, match="no usable sm_100 CUDA device|CUDA"):
        GpuHierRep(op)
    assert np.isfinite(op.blob).all()


def _malformed(mut):
    import copy
    from golden_io import load_golden
    op, _, _ = load_golden("g2d_log_h2plusH")
    op = copy.copy(op)
    op.channels = [copy.copy(ch) for ch in op.channels]
    mut(op)
    return op


@pytest.mark.parametrize("what,mut", [
    ("r_in length", lambda op: setattr(op.channels[0], "r_in", op.channels[0].r_in[:-1])),
    ("p2m_off length", lambda op: setattr(op.channels[0], "p2m_off", op.channels[0].p2m_off[:3])),
    ("m2l_src entry", lambda op: op.channels[0].m2l_src.__setitem__(0, op.n_clusters)),
    ("blr_src entry", lambda op: setattr(op, "blr_src", np.r_[-1, op.blr_src[1:]].astype(np.int32))),
    ("blr nnz", lambda op: setattr(op, "blr_rank", op.blr_rank[:-1])),
    ("near nnz", lambda op: setattr(op, "near_off", op.near_off[:-1])),
    ("near_src entry", lambda op: setattr(op, "near_src", op.near_src + op.n_clusters)),
    ("row pointer", lambda op: setattr(op, "near_rowptr", op.near_rowptr[::-1].copy())),
])
def test_validate_rejects_malformed_exports(what, mut):
    """The C side takes raw pointers without lengths, so every per-cluster
    array, per-entry array and source index is checked on the host first."""
    op = _malformed(mut)
    with pytest.raises(ValueError, match="bad export"):
        op.validate()
