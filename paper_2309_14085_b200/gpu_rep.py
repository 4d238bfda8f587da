"""GpuHierRep — drop-in GPU operator for the reference ``HierRep``.

Mirrors the reference's operator contract (engine.py:250-269, SURVEY.md
§8(b)):

* ``matvec(q)`` takes a 1-D vector of length N in the original point order
  (numpy array, list, or a torch CUDA tensor), never mutates it, returns a
  freshly allocated ``phi`` of dtype ``result_type(q, float64)``;
* ``ValueError("vector length mismatch")`` on a wrong length
  (engine.py:253-254), ``ValueError`` for a 2-D argument (the reference
  fails with a numpy broadcast ValueError there);
* repeated calls are bitwise identical (no atomics on the device);
* ``mem_scalars`` is the reference's own storage tally.

Extras: ``matmat(Q)`` for an N x k block (the reference's equivalent is a
column loop), numpy and torch-CUDA inputs, complex ``q`` with a real kernel
(two real products, as numpy would promote).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .packed import PackedOperator


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _desc_from_packed(op: PackedOperator, recompute: str = "", m2l_share: float = 1.0):
    """Build the h2g_export_desc; returns (desc, keepalive list).

    ``recompute``: comma list of block kinds evaluated from point
    coordinates even where they are stored ("near", "m2l"); blocks exported
    with offset -1 are always evaluated.  ``m2l_share`` in (0, 1): the share
    of the M2L work evaluated while the rest streams concurrently."""
    keep = []

    def arr(a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        keep.append(a)
        return a

    def i64(a):
        return _ptr(arr(a, np.int64), C.c_int64)

    def i32(a):
        return _ptr(arr(a, np.int32), C.c_int32)

    d = _lib.ExportDesc()
    d.abi_version = _lib.H2G_ABI_VERSION
    d.dim = op.dim
    d.kappa = op.kappa
    d.n_channels = len(op.channels)
    d.n_points = op.N
    d.n_clusters = op.n_clusters
    d.mem_scalars = int(op.mem_scalars)
    d.perm = i64(op.perm)
    d.level_offset = i64(op.level_offset)
    d.cl_start = i64(op.cl_start)
    d.cl_end = i64(op.cl_end)
    for i, ch in enumerate(op.channels):
        cd = d.channels[i]
        cd.r_in = i32(ch.r_in)
        cd.r_out = i32(ch.r_out)
        cd.p2m_off = i64(ch.p2m_off)
        cd.l2p_off = i64(ch.l2p_off)
        cd.m2m_off = i64(ch.m2m_off)
        cd.l2l_off = i64(ch.l2l_off)
        cd.m2l_rowptr = i64(ch.m2l_rowptr)
        cd.m2l_src = i32(ch.m2l_src)
        cd.m2l_off = i64(ch.m2l_off)
    d.blr_rowptr = i64(op.blr_rowptr)
    d.blr_src = i32(op.blr_src)
    d.blr_rank = i32(op.blr_rank)
    d.blr_u_off = i64(op.blr_u_off)
    d.blr_v_off = i64(op.blr_v_off)
    d.near_rowptr = i64(op.near_rowptr)
    d.near_src = i32(op.near_src)
    d.near_off = i64(op.near_off)
    blob = arr(op.blob, np.float64)
    d.blob_len = blob.size
    d.blob = _ptr(blob, C.c_double)
    # kernel-evaluation path (ABI 3): points, kernel rules, pivots
    for i, ch in enumerate(op.channels):
        if ch.has_pivots:
            cd = d.channels[i]
            cd.piv_in_ptr = i64(ch.piv_in_ptr)
            cd.piv_in = i64(ch.piv_in)
            cd.piv_out_ptr = i64(ch.piv_out_ptr)
            cd.piv_out = i64(ch.piv_out)
    if op.points_tree is not None:
        d.points_tree = _ptr(arr(op.points_tree, np.float64), C.c_double)
    kern = op.kernel or {}
    d.kernel_type = _lib.H2G_KERNELS.get(kern.get("name"), -1)
    d.has_diag = kern.get("diag") is not None
    d.zero_value = float(kern.get("zero_value", 0.0) or 0.0)
    d.diag = float(kern.get("diag") or 0.0)
    d.shift = float(kern.get("shift", 0.0) or 0.0)
    d.sigma = float(kern.get("sigma") or 0.0)
    mask = 0
    for part in (recompute or "").replace(" ", "").split(","):
        if part == "near":
            mask |= _lib.H2G_RECOMPUTE_NEAR
        elif part == "m2l":
            mask |= _lib.H2G_RECOMPUTE_M2L
        elif part:
            raise ValueError(f"recompute: unknown block kind {part!r} (near, m2l)")
    d.recompute = mask
    d.m2l_recompute_share = float(m2l_share)
    return d, keep


def _torch():
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    return torch


class GpuHierRep:
    """The operator of one reference ``HierRep``, resident on a B200."""

    def __init__(self, op: PackedOperator, device: int = 0, lib=None, recompute: str = "",
                 m2l_share: float = 1.0):
        L = lib or _lib.load()
        op.validate()
        desc, keep = _desc_from_packed(op, recompute, m2l_share)
        plan = C.c_void_p()
        _lib.check(L.h2g_plan_create(C.byref(desc), int(device), C.byref(plan)),
                   "h2g_plan_create")
        del keep
        self._L = L
        self._plan = plan
        self.device = int(device)
        self.N = int(op.N)
        self.variant = op.variant
        self.kernel = dict(op.kernel)
        self.mem_scalars = int(op.mem_scalars)
        self.kappa = op.kappa
        self.dim = op.dim

    # ------------------------------------------------------------ factories
    @classmethod
    def from_rep(cls, rep, device: int = 0, recompute: str = "") -> "GpuHierRep":
        """Export a reference HierRep (engine.py:235-269) and upload it.

        ``recompute`` ("near", "m2l" or both): those raw kernel blocks are
        evaluated on the device from the points and NCA pivots instead of
        streamed, and are not even exported (the reference's own
        store_near=False path, engine.py:260-268, extended to M2L =
        K[t_i, s_o], engine.py:176-179)."""
        from .export import export_rep
        kinds = {k for k in (recompute or "").replace(" ", "").split(",") if k}
        store = ",".join(k for k in ("near", "m2l") if k not in kinds)
        op = export_rep(rep, with_points=bool(kinds), store=store)
        return cls(op, device, recompute=",".join(sorted(kinds)))

    @classmethod
    def load(cls, path: str, device: int = 0) -> "GpuHierRep":
        return cls(PackedOperator.load(path), device)

    # ------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "_plan", None) is not None and self._plan.value:
            self._L.h2g_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --------------------------------------------------------------- stats
    def stats(self) -> dict:
        s = _lib.PlanStats()
        _lib.check(self._L.h2g_plan_get_stats(self._plan, C.byref(s)), "h2g_plan_get_stats")
        return {f: getattr(s, f) for f, _ in _lib.PlanStats._fields_}

    @property
    def alg_bytes(self) -> int:
        """Algorithmic bytes of one single-RHS matvec, 8*S + 16*N."""
        return 8 * self.mem_scalars + 16 * self.N

    def launches_per_matvec(self, nrhs: int = 1) -> int:
        return int(self._L.h2g_launches_per_matvec(self._plan, int(nrhs)))

    # -------------------------------------------------------------- apply
    def _apply_host(self, Q: np.ndarray, out: np.ndarray = None) -> np.ndarray:
        """Q: (N,) or (N, k) float64 -> same shape (into ``out`` if given)."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        k = 1 if Q.ndim == 1 else Q.shape[1]
        if out is None:
            out = np.empty_like(Q)
        elif (out.shape != Q.shape or out.dtype != np.float64
              or not out.flags.c_contiguous or not out.flags.writeable):
            raise ValueError("out must be a writable C-contiguous float64 array shaped like q")
        if Q.size == 0:
            return out
        _lib.check(self._L.h2g_matvec_host(self._plan, _ptr(Q, C.c_double), _ptr(out, C.c_double),
                                           self.N, k, k), "h2g_matvec_host")
        return out

    def _apply_torch(self, Q):
        torch = _torch()
        if Q.device.type != "cuda":
            raise ValueError("torch tensors must live on a CUDA device")
        if Q.device.index not in (None, self.device):
            raise ValueError(f"tensor on cuda:{Q.device.index}, operator on cuda:{self.device}")
        Q = Q.to(torch.float64).contiguous()
        k = 1 if Q.dim() == 1 else Q.shape[1]
        out = torch.empty_like(Q)
        stream = torch.cuda.current_stream(Q.device).cuda_stream
        _lib.check(self._L.h2g_matvec(self._plan, C.c_void_p(Q.data_ptr()),
                                      C.c_void_p(out.data_ptr()), self.N, k, k,
                                      C.c_void_p(stream)), "h2g_matvec")
        return out

    def _is_torch(self, q) -> bool:
        torch = _torch()
        return torch is not None and isinstance(q, torch.Tensor)

    def matvec(self, q, out=None):
        """phi = K~ q (HierRep.matvec, engine.py:250-269).

        ``out`` (numpy only, optional): a float64 array to receive phi, e.g. a
        pinned buffer for full-bandwidth device->host copies; returned."""
        if self._is_torch(q):
            if q.dim() != 1:
                raise ValueError("matvec expects a 1-D vector (use matmat for blocks)")
            if q.shape[0] != self.N:
                raise ValueError("vector length mismatch")
            if q.is_complex():
                return torch_complex(self._apply_torch(q.real), self._apply_torch(q.imag))
            return self._apply_torch(q)
        q = np.asarray(q)
        if q.ndim != 1:
            if q.ndim == 0 or len(q) != self.N:
                raise ValueError("vector length mismatch")
            raise ValueError("matvec expects a 1-D vector (use matmat for blocks)")
        if len(q) != self.N:
            raise ValueError("vector length mismatch")
        if np.iscomplexobj(q):
            if out is not None:
                raise ValueError("out= is not supported for complex q")
            return self._apply_host(q.real) + 1j * self._apply_host(q.imag)
        return self._apply_host(q, out)

    def matmat(self, Q):
        """Phi = K~ Q for an N x k block (reference: a column loop of matvec)."""
        if self._is_torch(Q):
            if Q.dim() != 2 or Q.shape[0] != self.N:
                raise ValueError("vector length mismatch")
            return self._apply_torch(Q)
        Q = np.asarray(Q)
        if Q.ndim != 2 or Q.shape[0] != self.N:
            raise ValueError("vector length mismatch")
        if np.iscomplexobj(Q):
            return self._apply_host(Q.real) + 1j * self._apply_host(Q.imag)
        return self._apply_host(Q)

    __call__ = matvec

    def profile_phases(self, q_dev, phi_dev, iters: int = 10):
        """Per-phase CUDA-event timing on the plan stream -> list of dicts."""
        cap = 64
        ms = (C.c_double * cap)()
        by = (C.c_int64 * cap)()
        names = (C.c_char_p * cap)()
        n = C.c_int()
        _lib.check(self._L.h2g_profile_phases(self._plan, C.c_void_p(q_dev.data_ptr()),
                                              C.c_void_p(phi_dev.data_ptr()), int(iters), ms, by,
                                              names, cap, C.byref(n)), "h2g_profile_phases")
        return [{"phase": names[i].decode(), "ms": ms[i], "bytes": int(by[i])}
                for i in range(n.value)]

    def profile_phases_batched(self, kb: int = 16, iters: int = 10):
        """Per-phase timing of one kb-wide pass of the batched-RHS engine."""
        cap = 64
        ms = (C.c_double * cap)()
        by = (C.c_int64 * cap)()
        names = (C.c_char_p * cap)()
        n = C.c_int()
        _lib.check(self._L.h2g_profile_phases_batched(self._plan, int(kb), int(iters), ms, by,
                                                      names, cap, C.byref(n)),
                   "h2g_profile_phases_batched")
        return [{"phase": names[i].decode(), "ms": ms[i], "bytes": int(by[i])}
                for i in range(n.value)]


def schedule_info(op: PackedOperator, n_sm: int = 148) -> dict:
    """Host-only view of the device schedule (phases, chunks, CTA balance)."""
    import json
    L = _lib.load()
    desc, keep = _desc_from_packed(op)
    buf = C.create_string_buffer(1 << 20)
    _lib.check(L.h2g_schedule_info(C.byref(desc), int(n_sm), buf, len(buf)), "h2g_schedule_info")
    del keep
    return json.loads(buf.value.decode())


def torch_complex(re, im):
    torch = _torch()
    return torch.complex(re, im)


def compute_potential(rep, q):
    """engine.py:321-322 for either a reference HierRep or a GpuHierRep."""
    return rep.matvec(q)
