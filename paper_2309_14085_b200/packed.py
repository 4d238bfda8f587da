"""Packed, level-major export of an H2* / (H2+H)* operator.

This is the single data format that crosses the drop-in boundary: the
exporter (:mod:`.export`, from a reference ``HierRep``), the native builder
(:mod:`.builder`) and the oracle (``oracle/packed_matvec.py``) all speak it,
and ``h2g_plan_create`` (include/h2g.h) consumes it through
:class:`h2g_export_desc`.

Layout (SURVEY.md §8(a')):

* ``perm[i]``: original point index of tree position ``i``; tree order is the
  concatenation of the leaf index sets in leaf-id (Z-order) order
  (reference tree.py:152-165).  Every cluster ``c`` is the contiguous slice
  ``[cl_start[c], cl_end[c])`` of tree order.
* cluster ids follow the reference: ``level_offset[l] + morton index``
  (tree.py:72-75), children of the cluster with in-level index ``m`` are
  ``m * 2**d + j`` (tree.py:176-178).
* every operator matrix lives in ONE fp64 ``blob``; matrix starts are aligned
  to :data:`ALIGN` doubles (32-byte sectors).  All matrices are stored
  **column-major** (columns contiguous) so that a warp whose lanes own rows
  reads each column with one coalesced request; the BLR ``V`` factor is kept
  row-major (``V^T`` column-major) for the same reason.
* per channel (reference NestedOperatorSet, engine.py:117-130):
  ``r_in / r_out`` per cluster; ``p2m_off`` / ``l2p_off`` per cluster
  (-1 = absent); ``m2m_off[c]`` holds m2m[(parent(c), c)] and ``l2l_off[c]``
  holds l2l[(c, parent(c))]; the M2L coupling is CSR by target cluster
  (``m2l_rowptr``, ``m2l_src`` ascending = lists_fn order, ``m2l_off``).
* BLR leg (blr.py:21-33): CSR by target cluster over the (X, Y) factors with
  rank > 0.  ``U`` (n_X x p) is stored LEAF-BLOCKED at ``blr_u_off``: for
  every leaf L inside X (tree order) the rows of L form one n_L x p
  column-major block starting at ``blr_u_off + (cl_start[L] - cl_start[X]) * p``,
  so each leaf's share of the factor is one contiguous run.  ``V`` (n_Y x p)
  is row-major at ``blr_v_off`` (= V^T column-major).
* near field (engine.py:260-268, 309-318): CSR by target leaf, dense
  n_X x n_Y column-major blocks at ``near_off``.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

SCHEMA = "h2g-export-2"
ALIGN = 1  # doubles: blocks are packed back to back (TMA bulk copies align down on device)

CHANNEL_FIELDS = ("r_in", "r_out", "p2m_off", "l2p_off", "m2m_off", "l2l_off",
                  "m2l_rowptr", "m2l_src", "m2l_off")
# NCA pivots (optional; the M2L kernel-evaluation path needs them)
PIVOT_FIELDS = ("piv_in_ptr", "piv_in", "piv_out_ptr", "piv_out")


@dataclass
class PackedChannel:
    r_in: np.ndarray       # int32[n_clusters]
    r_out: np.ndarray      # int32[n_clusters]
    p2m_off: np.ndarray    # int64[n_clusters]  r_out x n_X   (leaves)
    l2p_off: np.ndarray    # int64[n_clusters]  n_X x r_in    (leaves)
    m2m_off: np.ndarray    # int64[n_clusters]  r_out(parent) x r_out(c), keyed by child c
    l2l_off: np.ndarray    # int64[n_clusters]  r_in(c) x r_in(parent), keyed by child c
    m2l_rowptr: np.ndarray  # int64[n_clusters + 1]
    m2l_src: np.ndarray    # int32[nnz]
    m2l_off: np.ndarray    # int64[nnz]  r_in(X) x r_out(Y); -1 = evaluated, K[t_i(X), s_o(Y)]
    # NCA pivots as TREE POSITIONS, CSR by cluster (PivotQuad.t_i / s_o,
    # lowrank.py:45-59); None when not exported
    piv_in_ptr: np.ndarray = None   # int64[n_clusters + 1]
    piv_in: np.ndarray = None       # int64[sum r_in]
    piv_out_ptr: np.ndarray = None  # int64[n_clusters + 1]
    piv_out: np.ndarray = None      # int64[sum r_out]

    @property
    def has_pivots(self) -> bool:
        return self.piv_in is not None and self.piv_out is not None


@dataclass
class PackedOperator:
    variant: str
    kernel: dict            # {"name", "zero_value", "diag", "shift"}
    eps_far: float
    eps_ver: float
    N: int
    dim: int
    kappa: int
    n_max: int
    perm: np.ndarray        # int64[N]
    level_offset: np.ndarray  # int64[kappa + 2]
    cl_start: np.ndarray    # int64[n_clusters]
    cl_end: np.ndarray      # int64[n_clusters]
    channels: list          # [PackedChannel]
    blr_rowptr: np.ndarray  # int64[n_clusters + 1]
    blr_src: np.ndarray     # int32[nnz]
    blr_rank: np.ndarray    # int32[nnz]
    blr_u_off: np.ndarray   # int64[nnz]
    blr_v_off: np.ndarray   # int64[nnz]
    near_rowptr: np.ndarray  # int64[n_clusters + 1]
    near_src: np.ndarray    # int32[nnz]
    near_off: np.ndarray    # int64[nnz]; -1 = evaluated (store_near=False)
    blob: np.ndarray        # float64[blob_len]
    mem_scalars: int
    points_tree: np.ndarray = None  # float64[N, d] (optional; recompute paths)
    meta: dict = field(default_factory=dict)

    # ------------------------------------------------------------------ shape
    @property
    def n_clusters(self) -> int:
        return int(self.level_offset[-1])

    @property
    def has_blr(self) -> bool:
        return len(self.blr_src) > 0 or self.variant in ("h2plusH-star", "hstar", "hstd")

    def level_range(self, level: int):
        return int(self.level_offset[level]), int(self.level_offset[level + 1])

    def size(self, cid) -> int:
        return int(self.cl_end[cid] - self.cl_start[cid])

    def parent(self, cid: int):
        """Parent id via the Z-order rule m -> m >> d (tree.py:176)."""
        lo = self.level_offset
        l = int(np.searchsorted(lo, cid, side="right")) - 1
        if l == 0:
            return None
        return int(lo[l - 1] + ((cid - lo[l]) >> self.dim))

    def children(self, cid: int):
        lo = self.level_offset
        l = int(np.searchsorted(lo, cid, side="right")) - 1
        if l >= self.kappa:
            return []
        m = cid - int(lo[l])
        base = int(lo[l + 1]) + (m << self.dim)
        return list(range(base, base + (1 << self.dim)))

    def mat(self, off: int, rows: int, cols: int) -> np.ndarray:
        """Column-major rows x cols view into the blob."""
        return self.blob[off:off + rows * cols].reshape(cols, rows).T

    def mat_rowmajor(self, off: int, rows: int, cols: int) -> np.ndarray:
        return self.blob[off:off + rows * cols].reshape(rows, cols)

    def leaves_of(self, cid: int):
        """Leaf ids inside cluster cid, in tree order."""
        lo = self.level_offset
        l = int(np.searchsorted(lo, cid, side="right")) - 1
        shift = self.dim * (self.kappa - l)
        first = int(lo[self.kappa]) + ((cid - int(lo[l])) << shift)
        return range(first, first + (1 << shift))

    def blr_U(self, k: int, x: int) -> np.ndarray:
        """Dense n_X x p U factor of BLR entry k (target x) from its leaf blocks."""
        p = int(self.blr_rank[k])
        base = int(self.blr_u_off[k])
        s0 = int(self.cl_start[x])
        parts = [self.mat(base + (int(self.cl_start[L]) - s0) * p, self.size(L), p)
                 for L in self.leaves_of(x) if self.size(L)]
        return np.concatenate(parts, axis=0) if parts else np.zeros((0, p))

    @property
    def operator_bytes(self) -> int:
        """Algorithmic operator bytes: 8 * mem_scalars."""
        return 8 * int(self.mem_scalars)

    def stored_scalars(self) -> int:
        """Scalars actually referenced by the packed layout (no padding)."""
        tot = 0
        lo = self.level_offset
        for ch in self.channels:
            for cid in range(self.n_clusters):
                n = self.size(cid)
                if ch.p2m_off[cid] >= 0:
                    tot += ch.r_out[cid] * n
                if ch.l2p_off[cid] >= 0:
                    tot += ch.r_in[cid] * n
                p = self.parent(cid)
                if p is not None:
                    if ch.m2m_off[cid] >= 0:
                        tot += ch.r_out[p] * ch.r_out[cid]
                    if ch.l2l_off[cid] >= 0:
                        tot += ch.r_in[cid] * ch.r_in[p]
            for x in range(self.n_clusters):
                for k in range(ch.m2l_rowptr[x], ch.m2l_rowptr[x + 1]):
                    tot += ch.r_in[x] * ch.r_out[ch.m2l_src[k]]
        for x in range(self.n_clusters):
            for k in range(self.blr_rowptr[x], self.blr_rowptr[x + 1]):
                tot += self.blr_rank[k] * (self.size(x) + self.size(self.blr_src[k]))
            for k in range(self.near_rowptr[x], self.near_rowptr[x + 1]):
                tot += self.size(x) * self.size(self.near_src[k])
        del lo
        return int(tot)

    def without_blocks(self, near: bool = True, m2l: bool = True) -> "PackedOperator":
        """Shallow copy whose near and/or M2L blocks are marked "not stored"
        (offset -1): the plan then evaluates them from points_tree / the
        pivots, as the reference does with store_near=False
        (engine.py:260-268).  The blob is shared, not compacted."""
        import copy
        op = copy.copy(self)
        if near:
            op.near_off = np.full_like(self.near_off, -1)
        if m2l:
            op.channels = [copy.copy(ch) for ch in self.channels]
            for ch in op.channels:
                ch.m2l_off = np.full_like(ch.m2l_off, -1)
        return op

    # ------------------------------------------------------------- validate
    def validate(self):
        """Structural checks; raises ValueError("bad export: ...")."""
        def bad(msg):
            raise ValueError(f"bad export: {msg}")
        nc = self.n_clusters
        if self.perm.shape != (self.N,):
            bad("perm length")
        if not np.array_equal(np.sort(self.perm), np.arange(self.N)):
            bad("perm is not a permutation")
        if len(self.level_offset) != self.kappa + 2:
            bad("level_offset length")
        if len(self.channels) > 2:
            bad("at most two nested channels")
        for arr, n in ((self.cl_start, nc), (self.cl_end, nc),
                       (self.blr_rowptr, nc + 1), (self.near_rowptr, nc + 1)):
            if len(arr) != n:
                bad("per-cluster array length")
        def csr_ok(rowptr, name):
            if rowptr[0] != 0 or (len(rowptr) > 1 and np.any(np.diff(rowptr) < 0)):
                bad(f"{name} row pointer not monotone from 0")

        def in_range(idx, name):
            if len(idx) and (idx.min() < 0 or idx.max() >= nc):
                bad(f"{name} entry out of [0, n_clusters)")

        for ch in self.channels:
            for f in CHANNEL_FIELDS:
                a = getattr(ch, f)
                if f in ("m2l_src", "m2l_off"):
                    continue
                want = nc + 1 if f == "m2l_rowptr" else nc
                if len(a) != want:
                    bad(f"{f} length")
            csr_ok(ch.m2l_rowptr, "m2l")
            if len(ch.m2l_src) != ch.m2l_rowptr[-1] or len(ch.m2l_off) != ch.m2l_rowptr[-1]:
                bad("m2l nnz")
            in_range(ch.m2l_src, "m2l_src")
            if np.any(ch.r_in < 0) or np.any(ch.r_out < 0):
                bad("negative rank")
            if ch.has_pivots:
                if len(ch.piv_in_ptr) != nc + 1 or len(ch.piv_out_ptr) != nc + 1:
                    bad("pivot CSR length")
                if (not np.array_equal(np.diff(ch.piv_in_ptr), ch.r_in)
                        or not np.array_equal(np.diff(ch.piv_out_ptr), ch.r_out)):
                    bad("pivot count != rank")
                for a in (ch.piv_in, ch.piv_out):
                    if len(a) and (a.min() < 0 or a.max() >= self.N):
                        bad("pivot out of range")
        if self.points_tree is not None and self.points_tree.shape != (self.N, self.dim):
            bad("points_tree shape")
        csr_ok(self.near_rowptr, "near")
        csr_ok(self.blr_rowptr, "blr")
        if len(self.near_src) != self.near_rowptr[-1] or len(self.near_off) != self.near_rowptr[-1]:
            bad("near nnz")
        nb = self.blr_rowptr[-1]
        if (len(self.blr_src) != nb or len(self.blr_rank) != nb or len(self.blr_u_off) != nb
                or len(self.blr_v_off) != nb):
            bad("blr nnz")
        in_range(self.near_src, "near_src")
        in_range(self.blr_src, "blr_src")
        if nb and self.blr_rank.min() < 1:
            bad("BLR factor of rank < 1")
        if self.blob.dtype != np.float64:
            bad("blob dtype")

    # ------------------------------------------------------------------- io
    def to_arrays(self) -> dict:
        out = {
            "schema": np.asarray(SCHEMA),
            "variant": np.asarray(self.variant),
            "kernel_name": np.asarray(self.kernel.get("name", "")),
            "kernel_params": np.asarray(
                [self.kernel.get("zero_value", 0.0),
                 np.nan if self.kernel.get("diag") is None else self.kernel["diag"],
                 self.kernel.get("shift", 0.0),
                 np.nan if self.kernel.get("sigma") is None else self.kernel["sigma"]],
                dtype=np.float64),
            "scalars": np.asarray([self.N, self.dim, self.kappa, self.n_max,
                                   self.mem_scalars, len(self.channels)],
                                  dtype=np.int64),
            "eps": np.asarray([self.eps_far, self.eps_ver], dtype=np.float64),
        }
        for f in ("perm", "level_offset", "cl_start", "cl_end", "blr_rowptr",
                  "blr_src", "blr_rank", "blr_u_off", "blr_v_off",
                  "near_rowptr", "near_src", "near_off", "blob"):
            out[f] = getattr(self, f)
        for i, ch in enumerate(self.channels):
            for f in CHANNEL_FIELDS:
                out[f"ch{i}_{f}"] = getattr(ch, f)
            if ch.has_pivots:
                for f in PIVOT_FIELDS:
                    out[f"ch{i}_{f}"] = getattr(ch, f)
        if self.points_tree is not None:
            out["points_tree"] = self.points_tree
        return out

    def save(self, path: str, compress: bool = False):
        (np.savez_compressed if compress else np.savez)(path, **self.to_arrays())

    @classmethod
    def from_arrays(cls, z) -> "PackedOperator":
        if str(z["schema"]) != SCHEMA:
            raise ValueError(f"bad export: schema {z['schema']!r} != {SCHEMA}")
        N, dim, kappa, n_max, mem, nch = (int(x) for x in z["scalars"])
        zv, dg, sh, sg = (float(x) for x in z["kernel_params"])
        chans = [PackedChannel(**{f: np.asarray(z[f"ch{i}_{f}"]) for f in CHANNEL_FIELDS},
                               **{f: np.asarray(z[f"ch{i}_{f}"]) for f in PIVOT_FIELDS
                                  if f"ch{i}_{f}" in z})
                 for i in range(nch)]
        pts = np.asarray(z["points_tree"]) if "points_tree" in z else None
        return cls(variant=str(z["variant"]),
                   kernel={"name": str(z["kernel_name"]), "zero_value": zv,
                           "diag": None if np.isnan(dg) else dg, "shift": sh,
                           "sigma": None if np.isnan(sg) else sg},
                   eps_far=float(z["eps"][0]), eps_ver=float(z["eps"][1]),
                   N=N, dim=dim, kappa=kappa, n_max=n_max,
                   perm=np.asarray(z["perm"]), level_offset=np.asarray(z["level_offset"]),
                   cl_start=np.asarray(z["cl_start"]), cl_end=np.asarray(z["cl_end"]),
                   channels=chans,
                   blr_rowptr=np.asarray(z["blr_rowptr"]), blr_src=np.asarray(z["blr_src"]),
                   blr_rank=np.asarray(z["blr_rank"]), blr_u_off=np.asarray(z["blr_u_off"]),
                   blr_v_off=np.asarray(z["blr_v_off"]),
                   near_rowptr=np.asarray(z["near_rowptr"]), near_src=np.asarray(z["near_src"]),
                   near_off=np.asarray(z["near_off"]), blob=np.asarray(z["blob"]),
                   mem_scalars=mem, points_tree=pts)

    @classmethod
    def load(cls, path: str) -> "PackedOperator":
        if os.path.isdir(path):
            return cls.load_dir(path)
        with np.load(path, allow_pickle=False) as z:
            return cls.from_arrays({k: z[k] for k in z.files})

    def save_dir(self, path: str):
        """Directory form of the export: one raw ``.npy`` per field, so a
        multi-GB operator (config 3: 90 GB) is written at disk speed and
        loaded memory-mapped (:meth:`load_dir`) instead of through a zip."""
        os.makedirs(path, exist_ok=True)
        for k, v in self.to_arrays().items():
            np.save(os.path.join(path, f"{k}.npy"), np.asarray(v), allow_pickle=False)

    @classmethod
    def load_dir(cls, path: str, mmap: bool = True) -> "PackedOperator":
        z = {}
        for f in sorted(os.listdir(path)):
            if f.endswith(".npy"):
                z[f[:-4]] = np.load(os.path.join(path, f), mmap_mode="r" if mmap else None,
                                    allow_pickle=False)
        return cls.from_arrays(z)


class BlobWriter:
    """Appends matrices to one aligned fp64 blob (column-major by default)."""

    def __init__(self):
        self._parts = []
        self._len = 0

    def put(self, M: np.ndarray, order: str = "F") -> int:
        M = np.asarray(M)
        if np.iscomplexobj(M):
            raise TypeError("complex operators are not supported by the fp64 GPU path")
        pad = (-self._len) % ALIGN
        if pad:
            self._parts.append(np.zeros(pad))
            self._len += pad
        off = self._len
        flat = np.asarray(M, dtype=np.float64).ravel(order=order)
        self._parts.append(flat)
        self._len += flat.size
        return off

    def put_raw(self, flat: np.ndarray) -> int:
        """Append a flat run with no alignment padding (continues the previous one)."""
        off = self._len
        flat = np.asarray(flat, dtype=np.float64)
        self._parts.append(flat)
        self._len += flat.size
        return off

    def finish(self) -> np.ndarray:
        # trailing slack so that rounded-up bulk copies never leave the blob
        self._parts.append(np.zeros(ALIGN * 4))
        return np.concatenate(self._parts) if self._parts else np.zeros(0)
