"""Exporter: reference ``HierRep`` -> :class:`PackedOperator`.

Walks the reference objects duck-typed (it never imports the reference
package), so any object with the reference's field names exports:

* tree: ``rep.tree.clusters[cid].index_set / children / parent``,
  ``rep.tree.level_offset``, ``rep.tree.kappa`` (tree.py:39-90)
* channels: ``rep.channels[i]`` = NestedOperatorSet with dicts
  ``p2m, m2m, m2l, l2l, l2p``, ``quads`` and ``lists_fn`` (engine.py:117-130)
* BLR leg: ``rep.blr_leg.factors[(X, Y)]`` = LowRankFactor(U, V) (blr.py:21-33,
  lowrank.py:25-42)
* near field: ``rep.near_pairs`` + ``rep.near_blocks`` (engine.py:246-247,
  309-318); blocks the reference evaluates lazily (``store_near=False``,
  engine.py:265-267) are materialised with the same ``rep.kernel.block``
  call the reference would make, so stored and lazy exports are identical.
"""

from __future__ import annotations

import numpy as np

from .packed import BlobWriter, PackedChannel, PackedOperator


def _kernel_info(kernel) -> dict:
    name = {"Log2D": "log2d", "InverseR": "lap3d", "Gaussian": "gaussian"}.get(
        type(kernel).__name__, type(kernel).__name__)
    return {"name": name,
            "zero_value": float(getattr(kernel, "zero_value", 0.0) or 0.0),
            "diag": getattr(kernel, "diag", None),
            "shift": float(getattr(kernel, "shift", 0.0) or 0.0),
            "sigma": getattr(kernel, "sigma", None)}


def tree_layout(tree):
    """perm / cl_start / cl_end from the reference tree (tree.py:152-169).

    Checks the contiguity fact: every cluster equals a slice
    of the leaf-order permutation."""
    clusters = tree.clusters
    lo = np.asarray(tree.level_offset, dtype=np.int64)
    kappa = int(tree.kappa)
    nc = int(lo[-1])
    leaves = clusters[lo[kappa]:lo[kappa + 1]]
    sizes = np.array([len(c.index_set) for c in leaves], dtype=np.int64)
    perm = (np.concatenate([np.asarray(c.index_set, dtype=np.int64) for c in leaves])
            if len(leaves) else np.zeros(0, np.int64))
    cl_start = np.zeros(nc, np.int64)
    cl_end = np.zeros(nc, np.int64)
    ends = np.cumsum(sizes)
    cl_start[lo[kappa]:] = ends - sizes
    cl_end[lo[kappa]:] = ends
    d = tree.dim
    for l in range(kappa - 1, -1, -1):
        for m in range(int(lo[l + 1] - lo[l])):
            cid = int(lo[l]) + m
            c0 = int(lo[l + 1]) + (m << d)
            c1 = c0 + (1 << d) - 1
            cl_start[cid] = cl_start[c0]
            cl_end[cid] = cl_end[c1]
    for c in clusters:
        s, e = cl_start[c.id], cl_end[c.id]
        if not np.array_equal(perm[s:e], np.asarray(c.index_set)):
            raise ValueError(f"cluster {c.id} is not a contiguous tree-order slice")
    return perm, lo, cl_start, cl_end


def export_channel(tree, ops, blob: BlobWriter, inv_perm=None,
                   store_m2l: bool = True) -> PackedChannel:
    """One NestedOperatorSet (engine.py:117-130).  With ``inv_perm`` (original
    index -> tree position) the NCA pivots t_i / s_o of every cluster
    (PivotQuad, lowrank.py:45-59) are exported too, as tree positions: the
    M2L blocks are exactly K[t_i(X), s_o(Y)] (engine.py:176-179), so the
    device can evaluate them instead of streaming them.  ``store_m2l=False``
    exports every M2L block with offset -1 (not stored: evaluated from the
    pivots; needs ``inv_perm``)."""
    nc = len(tree.clusters)
    quads = ops.quads
    r_in = np.zeros(nc, np.int32)
    r_out = np.zeros(nc, np.int32)
    for cid, q in enumerate(quads):
        if q is not None:
            r_in[cid] = q.rank_in
            r_out[cid] = q.rank_out
    p2m_off = np.full(nc, -1, np.int64)
    l2p_off = np.full(nc, -1, np.int64)
    m2m_off = np.full(nc, -1, np.int64)
    l2l_off = np.full(nc, -1, np.int64)
    for cid, M in ops.p2m.items():
        p2m_off[cid] = blob.put(M)
    for cid, M in ops.l2p.items():
        l2p_off[cid] = blob.put(M)
    for (X, c), M in ops.m2m.items():
        if tree.clusters[c].parent != X:
            raise ValueError("m2m key is not (parent, child)")
        m2m_off[c] = blob.put(M)
    for (c, X), M in ops.l2l.items():
        if tree.clusters[c].parent != X:
            raise ValueError("l2l key is not (child, parent)")
        l2l_off[c] = blob.put(M)
    rowptr = np.zeros(nc + 1, np.int64)
    src, offs = [], []
    for X in range(nc):
        # same traversal as _channel_mvp (engine.py:216-219): lists_fn order,
        # only pairs that carry an operator
        for y in ops.lists_fn(X):
            M = ops.m2l.get((X, y))
            if M is None:
                continue
            src.append(y)
            offs.append(blob.put(M) if store_m2l else -1)
        rowptr[X + 1] = len(src)
    piv = {}
    if inv_perm is not None:
        for name, attr in (("in", "t_i"), ("out", "s_o")):
            ptr = np.zeros(nc + 1, np.int64)
            idx = []
            for cid, q in enumerate(quads):
                if q is not None and not q.empty:
                    ids = np.asarray(getattr(q, attr), dtype=np.int64)
                    idx.append(inv_perm[ids])
                    ptr[cid + 1] = len(ids)
            piv[f"piv_{name}_ptr"] = np.cumsum(ptr)
            piv[f"piv_{name}"] = (np.concatenate(idx) if idx else np.zeros(0)).astype(np.int64)
    return PackedChannel(r_in=r_in, r_out=r_out, p2m_off=p2m_off, l2p_off=l2p_off,
                         m2m_off=m2m_off, l2l_off=l2l_off, m2l_rowptr=rowptr,
                         m2l_src=np.asarray(src, np.int32),
                         m2l_off=np.asarray(offs, np.int64), **piv)


def _put_leaf_blocked(blob: BlobWriter, U, tree, X: int) -> int:
    """U (n_X x p) as consecutive column-major blocks, one per leaf of X in
    tree order (packed.py: BLR leg layout).  Returns the first offset."""
    U = np.asarray(U)
    lo = tree.level_offset
    l = tree.clusters[X].level
    kappa, d = tree.kappa, tree.dim
    shift = d * (kappa - l)
    first = lo[kappa] + ((X - lo[l]) << shift)
    r0, off0 = 0, None
    for L in range(first, first + (1 << shift)):
        n = len(tree.clusters[L].index_set)
        if n == 0:
            continue
        off = blob.put_raw(np.asarray(U[r0:r0 + n], dtype=np.float64).ravel(order="F"))
        off0 = off if off0 is None else off0
        r0 += n
    if off0 is None:
        off0 = blob.put_raw(np.zeros(0))
    return off0


def export_rep(rep, with_points: bool = True, store: str = "near,m2l") -> PackedOperator:
    """Pack a reference ``HierRep`` (engine.py:235-269) for the GPU plan.

    ``store`` names the raw kernel blocks written to the blob ("near",
    "m2l"); the others are exported with offset -1 and evaluated on the
    device from the points and NCA pivots (M2L = K[t_i(X), s_o(Y)],
    engine.py:176-179; near = K[t^X, t^Y], the reference's own
    store_near=False path, engine.py:260-268).  Leaving a kind out needs
    ``with_points``."""
    kinds = {k for k in store.replace(" ", "").split(",") if k}
    if kinds - {"near", "m2l"}:
        raise ValueError(f"store: unknown block kinds {sorted(kinds - {'near', 'm2l'})}")
    if kinds != {"near", "m2l"} and not with_points:
        raise ValueError("blocks that are not stored are evaluated from points: with_points=True")
    tree = rep.tree
    kernel = rep.kernel
    if np.issubdtype(np.dtype(getattr(kernel, "dtype", np.float64)), np.complexfloating):
        raise TypeError("complex kernels are not supported by the fp64 GPU path")
    perm, lo, cl_start, cl_end = tree_layout(tree)
    nc = int(lo[-1])
    blob = BlobWriter()
    inv_perm = np.empty_like(perm)
    inv_perm[perm] = np.arange(len(perm))
    channels = [export_channel(tree, ops, blob, inv_perm, store_m2l="m2l" in kinds)
                for ops in rep.channels]

    # BLR leg: factor dict is level-major / X asc / Y asc (blr.py:53-59);
    # rank-0 factors are skipped exactly as mvp_blr does (blr.py:79-80)
    blr_rowptr = np.zeros(nc + 1, np.int64)
    b_src, b_rank, b_u, b_v = [], [], [], []
    if rep.blr_leg is not None:
        if getattr(rep.blr_leg, "near_pairs", None):
            raise ValueError("BLR leg with its own near field is not a hot-path variant")
        by_x = {}
        for (x, y), f in rep.blr_leg.factors.items():
            if f.rank == 0:
                continue
            by_x.setdefault(x, []).append((y, f))
        for X in range(nc):
            for y, f in by_x.get(X, []):
                b_src.append(y)
                b_rank.append(f.rank)
                b_u.append(_put_leaf_blocked(blob, f.U, tree, X))  # leaf-blocked U
                b_v.append(blob.put(np.conj(f.V), order="C"))  # n_Y x p, row-major
            blr_rowptr[X + 1] = len(b_src)

    # near field: pairs in (leaf X asc, Y asc) order (engine.py:309-314)
    near_rowptr = np.zeros(nc + 1, np.int64)
    n_src, n_off = [], []
    pairs_by_x = {}
    for x, y in rep.near_pairs:
        pairs_by_x.setdefault(x, []).append(y)
    for X in range(nc):
        for y in pairs_by_x.get(X, []):
            t = tree.clusters[X].index_set
            s = tree.clusters[y].index_set
            if len(t) == 0 or len(s) == 0:
                continue  # engine.py:263-264
            n_src.append(y)
            if "near" not in kinds:
                n_off.append(-1)
                continue
            blk = rep.near_blocks.get((X, y))
            if blk is None:
                blk = kernel.block(t, s)  # the reference's lazy path
            n_off.append(blob.put(blk))
        near_rowptr[X + 1] = len(n_src)

    pts = None
    if with_points:
        pts = np.ascontiguousarray(tree.particles.points[perm], dtype=np.float64)
    out = PackedOperator(
        variant=rep.variant, kernel=_kernel_info(kernel),
        eps_far=float(rep.eps_far), eps_ver=float(rep.eps_ver),
        N=int(tree.particles.N), dim=int(tree.dim), kappa=int(tree.kappa),
        n_max=int(tree.n_max), perm=perm, level_offset=lo,
        cl_start=cl_start, cl_end=cl_end, channels=channels,
        blr_rowptr=blr_rowptr, blr_src=np.asarray(b_src, np.int32),
        blr_rank=np.asarray(b_rank, np.int32), blr_u_off=np.asarray(b_u, np.int64),
        blr_v_off=np.asarray(b_v, np.int64), near_rowptr=near_rowptr,
        near_src=np.asarray(n_src, np.int32), near_off=np.asarray(n_off, np.int64),
        blob=blob.finish(), mem_scalars=int(rep.mem_scalars), points_tree=pts,
        meta={"source": "reference HierRep"})
    out.validate()
    return out
