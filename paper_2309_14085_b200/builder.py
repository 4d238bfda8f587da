"""Native operator builder (libh2b.so, include/h2b.h) -> PackedOperator.

``build_variant`` mirrors the reference entry point of the same name
(engine.py:325-373) for the two hot-path variants, taking the point cloud
and the kernel by name (the reference takes a ClusterTree and a Kernel
object built from the same points, tree.py:111 / kernels.py:211):

    op = build_variant("h2star-bt", points, kernel="log2d", n_max=64, eps=1e-8)
    rep = GpuHierRep(op)          # drop-in matvec

Kernels: "log2d" (Log2D, kernels.py:63-71), "lap3d" (InverseR,
kernels.py:74-81) and "gaussian" (config 4's exp(-r^2/(2 sigma^2)) with
r=0 -> 1 and a 1e-6 diagonal shift, added via the Kernel hook).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .packed import CHANNEL_FIELDS, PIVOT_FIELDS, PackedChannel, PackedOperator

LIBDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
VARIANTS = {"h2star-bt": 0, "h2plusH-star": 1}
KERNELS = {"log2d": 0, "lap3d": 1, "gaussian": 2}
# reference defaults (kernels.py:63-81 + the cfg-4 Gaussian)
KERNEL_DEFAULTS = {
    "log2d": {"zero_value": 0.0, "diag": None, "shift": 0.0, "sigma": None},
    "lap3d": {"zero_value": 0.0, "diag": None, "shift": 0.0, "sigma": None},
    "gaussian": {"zero_value": 1.0, "diag": None, "shift": 1e-6, "sigma": 0.1},
}


class H2bParams(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("dim", C.c_int32), ("n_points", C.c_int64),
                ("points", C.POINTER(C.c_double)), ("n_max", C.c_int32), ("variant", C.c_int32),
                ("kernel", C.c_int32), ("has_diag", C.c_int32), ("zero_value", C.c_double),
                ("diag", C.c_double), ("shift", C.c_double), ("sigma", C.c_double),
                ("eps_far", C.c_double), ("eps_ver", C.c_double), ("n_threads", C.c_int32),
                ("skip_blocks", C.c_int32)]


class H2bFillChannel(C.Structure):
    _fields_ = [("r_in", C.POINTER(C.c_int32)), ("r_out", C.POINTER(C.c_int32)),
                ("m2l_rowptr", C.POINTER(C.c_int64)), ("m2l_src", C.POINTER(C.c_int32)),
                ("m2l_off", C.POINTER(C.c_int64)), ("piv_in_ptr", C.POINTER(C.c_int64)),
                ("piv_in", C.POINTER(C.c_int64)), ("piv_out_ptr", C.POINTER(C.c_int64)),
                ("piv_out", C.POINTER(C.c_int64))]


class H2bFillDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("kernel", C.c_int32), ("has_diag", C.c_int32),
                ("n_channels", C.c_int32), ("n_points", C.c_int64), ("n_clusters", C.c_int64),
                ("points_tree", C.POINTER(C.c_double)), ("zero_value", C.c_double),
                ("diag", C.c_double), ("shift", C.c_double), ("sigma", C.c_double),
                ("cl_start", C.POINTER(C.c_int64)), ("cl_end", C.POINTER(C.c_int64)),
                ("near_rowptr", C.POINTER(C.c_int64)), ("near_src", C.POINTER(C.c_int32)),
                ("near_off", C.POINTER(C.c_int64)), ("channels", H2bFillChannel * 2),
                ("n_threads", C.c_int32), ("pad", C.c_int32)]


H2B_SYMBOLS = ("h2b_build", "h2b_get_array", "h2b_get_scalar", "h2b_get_timing", "h2b_free",
               "h2b_last_error", "h2b_abi_version", "h2b_fill_kernel_blocks")
_LIB = None


def load():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(LIBDIR, "libh2b.so")
    if not os.path.exists(path):
        raise RuntimeError(f"native builder {path} is missing; run "
                           "`python -m paper_2309_14085_b200.build`")
    L = C.CDLL(path)
    L.h2b_build.argtypes = [C.POINTER(H2bParams), C.POINTER(C.c_void_p)]
    L.h2b_get_array.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p),
                                C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    L.h2b_get_scalar.argtypes = [C.c_void_p, C.c_char_p]
    L.h2b_get_scalar.restype = C.c_int64
    L.h2b_get_timing.argtypes = [C.c_void_p, C.c_char_p]
    L.h2b_get_timing.restype = C.c_double
    L.h2b_free.argtypes = [C.c_void_p]
    L.h2b_fill_kernel_blocks.argtypes = [C.POINTER(H2bFillDesc), C.POINTER(C.c_double), C.c_int64]
    L.h2b_last_error.restype = C.c_char_p
    if L.h2b_abi_version() != 1:
        raise RuntimeError("libh2b.so ABI mismatch; rebuild")
    _LIB = L
    return L


_DT = {0: np.int32, 1: np.int64, 2: np.float64}


class _Result:
    """Owns an h2b_result; arrays are zero-copy views kept alive by it."""

    def __init__(self, L, handle):
        self._L = L
        self.h = handle

    def array(self, name, copy=True):
        ptr, n, dt = C.c_void_p(), C.c_int64(), C.c_int32()
        rc = self._L.h2b_get_array(self.h, name.encode(), C.byref(ptr), C.byref(n), C.byref(dt))
        if rc:
            raise KeyError(name)
        dtype = np.dtype(_DT[dt.value])
        if n.value == 0:
            return np.zeros(0, dtype)
        buf = (C.c_char * (n.value * dtype.itemsize)).from_address(ptr.value)
        a = np.frombuffer(buf, dtype=dtype, count=n.value)
        return a.copy() if copy else a

    def scalar(self, name):
        return int(self._L.h2b_get_scalar(self.h, name.encode()))

    def timing(self, name):
        return float(self._L.h2b_get_timing(self.h, name.encode()))

    def __del__(self):
        if self.h:
            self._L.h2b_free(self.h)
            self.h = None


def build_variant(variant: str, points, kernel: str = "log2d", n_max: int = 64,
                  eps: float = 1e-8, eps_far: float = None, eps_ver: float = None,
                  n_threads: int = 0, zero_value=None, diag=None, shift=None, sigma=None,
                  copy_blob: bool = False, store: str = "near,m2l") -> PackedOperator:
    """Native build_variant (engine.py:325-373) -> PackedOperator.

    ``store`` names the raw kernel blocks kept in the blob ("near", "m2l");
    the others are exported with offset -1 and evaluated on the device from
    the points / NCA pivots (the reference's store_near=False,
    engine.py:260-268, extended to M2L = K[t_i, s_o], engine.py:176-179).
    The pivots are always exported."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant '{variant}'")
    if kernel not in KERNELS:
        raise ValueError(f"unknown kernel '{kernel}'")
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] not in (1, 2, 3) or len(pts) == 0:
        raise ValueError("points must be a non-empty (N, d) array, d in 1..3")
    kd = dict(KERNEL_DEFAULTS[kernel])
    for k, v in (("zero_value", zero_value), ("diag", diag), ("shift", shift), ("sigma", sigma)):
        if v is not None:
            kd[k] = v
    eps_far = eps if eps_far is None else eps_far
    eps_ver = eps if eps_ver is None else eps_ver
    L = load()
    p = H2bParams()
    p.abi_version = 1
    p.dim = pts.shape[1]
    p.n_points = len(pts)
    p.points = pts.ctypes.data_as(C.POINTER(C.c_double))
    p.n_max = int(n_max)
    p.variant = VARIANTS[variant]
    p.kernel = KERNELS[kernel]
    p.has_diag = kd["diag"] is not None
    p.zero_value = float(kd["zero_value"])
    p.diag = float(kd["diag"] or 0.0)
    p.shift = float(kd["shift"])
    p.sigma = float(kd["sigma"] or 0.1)
    p.eps_far = float(eps_far)
    p.eps_ver = float(eps_ver)
    p.n_threads = int(n_threads)
    kinds = {k for k in store.replace(" ", "").split(",") if k}
    if kinds - {"near", "m2l"}:
        raise ValueError(f"store: unknown block kinds {sorted(kinds - {'near', 'm2l'})}")
    p.skip_blocks = (0 if "near" in kinds else 1) | (0 if "m2l" in kinds else 2)
    h = C.c_void_p()
    rc = L.h2b_build(C.byref(p), C.byref(h))
    if rc:
        msg = L.h2b_last_error().decode()
        if rc == 2:
            raise ArithmeticError(f"SingularCrossMatrix: {msg}")
        raise RuntimeError(f"h2b_build failed ({rc}): {msg}")
    R = _Result(L, h)
    nch = R.scalar("n_channels")
    chans = [PackedChannel(**{f: R.array(f"ch{i}_{f}") for f in CHANNEL_FIELDS},
                           **{f: R.array(f"ch{i}_{f}") for f in PIVOT_FIELDS})
             for i in range(nch)]
    blob = R.array("blob", copy=copy_blob)
    op = PackedOperator(
        variant=variant, kernel={"name": kernel, **kd}, eps_far=float(eps_far),
        eps_ver=float(eps_ver), N=len(pts), dim=pts.shape[1], kappa=R.scalar("kappa"),
        n_max=int(n_max), perm=R.array("perm"), level_offset=R.array("level_offset"),
        cl_start=R.array("cl_start"), cl_end=R.array("cl_end"), channels=chans,
        blr_rowptr=R.array("blr_rowptr"), blr_src=R.array("blr_src"),
        blr_rank=R.array("blr_rank"), blr_u_off=R.array("blr_u_off"),
        blr_v_off=R.array("blr_v_off"), near_rowptr=R.array("near_rowptr"),
        near_src=R.array("near_src"), near_off=R.array("near_off"), blob=blob,
        mem_scalars=R.scalar("mem_scalars"),
        points_tree=R.array("points_tree").reshape(len(pts), pts.shape[1]),
        meta={"source": "native builder (libh2b.so)",
              "build_s": {k: R.timing(k) for k in ("tree", "partition", "pivots", "operators",
                                                    "blr", "near", "total")}})
    if not copy_blob:
        op.meta["_keepalive"] = R  # blob is a view into the native result
    op.validate()
    return op


def materialize_blocks(op: PackedOperator, near: bool = True, m2l: bool = True,
                       n_threads: int = 0) -> PackedOperator:
    """A copy of ``op`` whose NOT-stored raw kernel blocks (offset -1: an
    export built with store="" or a compact fixture) are evaluated into the
    blob by the native builder (h2b_fill_kernel_blocks, include/h2b.h):
    M2L = K[t_i(X), s_o(Y)] (engine.py:176-179) in target-major order (each
    target's row contiguous, as a stored build lays it out), near = K[t^X,
    t^Y] (engine.py:309-318) leaf by leaf.  Bitwise the blocks a stored
    build holds; seconds instead of the NCA pivot search."""
    import copy
    L = load()
    kname = op.kernel.get("name")
    if kname not in KERNELS or op.points_tree is None:
        raise ValueError("materialize_blocks needs points_tree and a known kernel")
    out = copy.copy(op)
    n = len(op.blob)
    keep = []

    def arr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a

    def p64(a):
        return arr(a, np.int64).ctypes.data_as(C.POINTER(C.c_int64))

    def p32(a):
        return arr(a, np.int32).ctypes.data_as(C.POINTER(C.c_int32))

    f = H2bFillDesc()
    f.dim, f.kernel, f.n_channels = op.dim, KERNELS[kname], len(op.channels)
    f.has_diag = op.kernel.get("diag") is not None
    f.n_points, f.n_clusters = op.N, op.n_clusters
    f.points_tree = arr(op.points_tree, np.float64).ctypes.data_as(C.POINTER(C.c_double))
    f.zero_value = float(op.kernel.get("zero_value") or 0.0)
    f.diag = float(op.kernel.get("diag") or 0.0)
    f.shift = float(op.kernel.get("shift") or 0.0)
    f.sigma = float(op.kernel.get("sigma") or 0.1)
    f.cl_start, f.cl_end = p64(op.cl_start), p64(op.cl_end)
    f.n_threads = int(n_threads)
    out.channels = []
    for i, ch in enumerate(op.channels):
        ch2 = copy.copy(ch)
        offs = np.full_like(ch.m2l_off, -1)
        if m2l:
            todo = np.flatnonzero(ch.m2l_off < 0)
            if len(todo):
                x = np.repeat(np.arange(op.n_clusters), np.diff(ch.m2l_rowptr))[todo]
                sz = ch.r_in[x].astype(np.int64) * ch.r_out[ch.m2l_src[todo]].astype(np.int64)
                offs[todo] = n + np.concatenate([[0], np.cumsum(sz)[:-1]])
                n += int(sz.sum())
        ch2.m2l_off = np.where(ch.m2l_off < 0, offs, ch.m2l_off)
        out.channels.append(ch2)
        c = f.channels[i]
        c.r_in, c.r_out = p32(ch.r_in), p32(ch.r_out)
        c.m2l_rowptr, c.m2l_src, c.m2l_off = p64(ch.m2l_rowptr), p32(ch.m2l_src), p64(offs)
        c.piv_in_ptr, c.piv_in = p64(ch.piv_in_ptr), p64(ch.piv_in)
        c.piv_out_ptr, c.piv_out = p64(ch.piv_out_ptr), p64(ch.piv_out)
    noffs = np.full_like(op.near_off, -1)
    if near:
        todo = np.flatnonzero(op.near_off < 0)
        if len(todo):
            x = np.repeat(np.arange(op.n_clusters), np.diff(op.near_rowptr))[todo]
            y = op.near_src[todo]
            sz = (op.cl_end[x] - op.cl_start[x]) * (op.cl_end[y] - op.cl_start[y])
            noffs[todo] = n + np.concatenate([[0], np.cumsum(sz)[:-1]])
            n += int(sz.sum())
    out.near_off = np.where(op.near_off < 0, noffs, op.near_off)
    f.near_rowptr, f.near_src, f.near_off = p64(op.near_rowptr), p32(op.near_src), p64(noffs)
    blob = np.empty(n + 4, dtype=np.float64)
    blob[:len(op.blob)] = op.blob
    blob[n:] = 0.0
    rc = L.h2b_fill_kernel_blocks(C.byref(f), blob.ctypes.data_as(C.POINTER(C.c_double)),
                                  len(blob))
    if rc:
        raise RuntimeError(f"h2b_fill_kernel_blocks failed ({rc}): {L.h2b_last_error().decode()}")
    del keep
    out.blob = blob
    out.meta = dict(op.meta)
    out.meta.pop("_keepalive", None)
    out.validate()
    return out


def uniform_points(N: int, d: int, seed: int = 42) -> np.ndarray:
    """Reference points.py:10-12 (default_rng(seed).uniform(-1, 1, (N, d)))."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(N, d))


def jittered_grid(n_side: int, d: int = 3, seed: int = 42) -> np.ndarray:
    """Config 5's jittered grid: cell centres -1 + (i + 0.5) h (as
    points.py:34-38's uniform_grid, tensor order 'ij') plus U(-h/2, h/2)
    per coordinate, h = 2 / n_side."""
    h = 2.0 / n_side
    axis = -1.0 + (np.arange(n_side) + 0.5) * h
    grids = np.meshgrid(*([axis] * d), indexing="ij")
    pts = np.stack([g.ravel() for g in grids], axis=1)
    rng = np.random.default_rng(seed)
    return pts + rng.uniform(-0.5 * h, 0.5 * h, size=pts.shape)
