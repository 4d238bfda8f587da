"""Loading helpers for the golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from paper_2309_14085_b200.packed import PackedOperator

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names():
    # operator fixtures (gmres_*.npz hold solver trajectories, not operators)
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "g*.npz"))
                  if not os.path.basename(p).startswith("gmres_"))


def load_golden(name):
    with np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"), allow_pickle=False) as z:
        arrays = {k: z[k] for k in z.files}
    op = PackedOperator.from_arrays(arrays)
    meta = json.loads(str(arrays["meta"]))
    return op, arrays, meta


def rel_err(a, b):
    """2-norm relative error (reference bench.py:100-104)."""
    den = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - b) / den) if den else float(np.linalg.norm(a))


def materialize(op):
    """A copy of ``op`` whose "not stored" blocks (offset -1: the compact
    fixtures, tests/golden/make_golden.py COMPACT) are evaluated into a new
    blob with the oracle's restatement of Kernel.block (kernels.py:36-57):
    M2L = K[t_i(X), s_o(Y)] (engine.py:176-179), near = K[t^X, t^Y]
    (engine.py:309-318).  The fixture's meta records how far these are from
    the reference's own stored blocks (blk_maxdiff_*)."""
    import copy
    from oracle.packed_matvec import kernel_block
    out = copy.copy(op)
    parts = [op.blob]
    n = len(op.blob)

    def put(M):
        nonlocal n
        flat = np.asarray(M, dtype=np.float64).ravel(order="F")
        parts.append(flat)
        n += flat.size
        return n - flat.size

    out.channels = []
    for ch in op.channels:
        ch2 = copy.copy(ch)
        offs = ch.m2l_off.copy()
        for X in range(op.n_clusters):
            ti = ch.piv_in[ch.piv_in_ptr[X]:ch.piv_in_ptr[X + 1]]
            for k in range(ch.m2l_rowptr[X], ch.m2l_rowptr[X + 1]):
                if offs[k] >= 0:
                    continue
                Y = ch.m2l_src[k]
                offs[k] = put(kernel_block(op, ti, ch.piv_out[ch.piv_out_ptr[Y]:ch.piv_out_ptr[Y + 1]]))
        ch2.m2l_off = offs
        out.channels.append(ch2)
    noff = op.near_off.copy()
    for X in range(op.n_clusters):
        for k in range(op.near_rowptr[X], op.near_rowptr[X + 1]):
            if noff[k] >= 0:
                continue
            Y = op.near_src[k]
            noff[k] = put(kernel_block(op, np.arange(op.cl_start[X], op.cl_end[X]),
                                       np.arange(op.cl_start[Y], op.cl_end[Y])))
    out.near_off = noff
    out.blob = np.concatenate(parts + [np.zeros(4)])
    out.validate()
    return out


def is_compact(op):
    return bool((op.near_off < 0).any() or any((ch.m2l_off < 0).any() for ch in op.channels))
