"""Multi-GPU matvec: subtree-sharded plans + one all-gather per matvec.

One process per GPU (``torch.distributed``, NCCL).  Rank r of R builds a
plan restricted to its subtrees (``h2g_plan_create_sharded``, include/h2g.h):
the Morton range [r*S/R, (r+1)*S/R) of the S subtrees at level L_s, the
replicated coarse levels, and the BLR V^T q pieces over its own rows.  q is
replicated.  A matvec is

    h2g_matvec_begin(q)        P2M, BLR pieces, M2M of the owned subtrees
    h2g_shard_pack(send)       owned multipole coefficients v (levels >= L_s)
                               + split-K partials of replicated BLR targets
    all_gather(send -> recv)   NCCL, max_send_slots doubles per rank
    h2g_shard_unpack(recv)
    h2g_matvec_end(phi)        coarse M2M, M2L/L2L, L2P + BLR U + near field:
                               phi rows [row_begin, row_end) of tree order

No reduction of phi is ever needed (rows are owned); ``gather_full=True``
combines the ranks' rows with one all-reduce (disjoint rows, exact).

``schedule_view`` exposes the same per-rank schedule to numpy; the test
infrastructure executes it on CPU (oracle/sched_emulator.py, gloo in
tests/test_sharded.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .gpu_rep import _desc_from_packed
from .packed import PackedOperator


class ShardedGpuHierRep:
    """Rank ``rank``'s share of one operator.  ``recompute`` ("near", "m2l")
    evaluates those raw kernel blocks on the device even where stored, as
    GpuHierRep does (blocks exported with offset -1 are always evaluated):
    config 5's operating mode, whose stored blocks would not fit."""

    def __init__(self, op: PackedOperator, rank: int, nranks: int, device: int = 0,
                 group=None, lib=None, recompute: str = "", m2l_share: float = 1.0):
        L = lib or _lib.load()
        op.validate()
        desc, keep = _desc_from_packed(op, recompute, m2l_share)
        plan = C.c_void_p()
        _lib.check(L.h2g_plan_create_sharded(C.byref(desc), int(device), int(rank), int(nranks),
                                             C.byref(plan)), "h2g_plan_create_sharded", L=L)
        del keep
        self._L, self._plan = L, plan
        self.rank, self.nranks, self.device, self.group = rank, nranks, device, group
        self.N = op.N
        self.mem_scalars = op.mem_scalars
        self.recompute = recompute
        info = _lib.ShardInfo()
        _lib.check(L.h2g_shard_get_info(plan, C.byref(info)), L=L)
        self.info = {f: getattr(info, f) for f, _ in _lib.ShardInfo._fields_}
        self._send = self._recv = None

    def launches_per_matvec(self) -> int:
        """gather + phases + scatter (h2g_launches_per_matvec) + pack + unpack."""
        return int(self._L.h2g_launches_per_matvec(self._plan, 1)) + (2 if self.nranks > 1 else 0)

    def close(self):
        if getattr(self, "_plan", None) is not None and self._plan.value:
            self._L.h2g_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the three halves (torch CUDA tensors, current stream) ---------------
    def _buffers(self, torch):
        if self._send is None:
            mx = max(1, self.info["max_send_slots"])
            dev = f"cuda:{self.device}"
            self._send = torch.zeros(mx, dtype=torch.float64, device=dev)
            self._recv = torch.zeros(mx * self.nranks, dtype=torch.float64, device=dev)
        return self._send, self._recv

    def begin(self, q, stream):
        _lib.check(self._L.h2g_matvec_begin(self._plan, C.c_void_p(q.data_ptr()), self.N,
                                            C.c_void_p(stream)), "h2g_matvec_begin", L=self._L)

    def pack(self, send, stream):
        _lib.check(self._L.h2g_shard_pack(self._plan, C.c_void_p(send.data_ptr()),
                                          C.c_void_p(stream)), L=self._L)

    def overlap(self, stream):
        """The owned near field (reads only q): launched after the all-gather
        has been started, it runs while the exchange is in flight."""
        _lib.check(self._L.h2g_shard_overlap(self._plan, C.c_void_p(stream)),
                   "h2g_shard_overlap", L=self._L)

    def _all_gather_overlapped(self, dist, recv, send, stream):
        """All-gather on NCCL's stream with the owned near field on ours."""
        work = dist.all_gather_into_tensor(recv, send, group=self.group, async_op=True)
        self.overlap(stream)
        work.wait()  # our stream waits for the exchange; the host does not block

    def unpack(self, recv, stream):
        _lib.check(self._L.h2g_shard_unpack(self._plan, C.c_void_p(recv.data_ptr()),
                                            C.c_void_p(stream)), L=self._L)

    def end(self, phi, stream):
        _lib.check(self._L.h2g_matvec_end(self._plan, C.c_void_p(phi.data_ptr()), self.N,
                                          C.c_void_p(stream)), "h2g_matvec_end", L=self._L)

    def owned_rows(self):
        """Tree-order rows [row_begin, row_end) this rank owns; their points are
        perm[row_begin:row_end] (the distributed-vector layout)."""
        return int(self.info["row_begin"]), int(self.info["row_end"])

    def matvec_distributed(self, q_own):
        """Distributed vectors: ``q_own`` = this rank's rows of q in tree order
        (q[perm[row_begin:row_end]]), no rank holds all of q.  The x halo
        (near-field and BLR sources of other ranks' rows) is all-gathered
        first, then the coefficient exchange as in :meth:`matvec`.  Returns
        this rank's rows of phi in tree order."""
        import torch
        import torch.distributed as dist
        rb, re_ = self.owned_rows()
        if q_own.shape[0] != re_ - rb:
            raise ValueError("vector length mismatch")
        q_own = q_own.to(torch.float64).contiguous()
        stream = torch.cuda.current_stream(q_own.device).cuda_stream
        L = self._L
        phi_own = torch.empty_like(q_own)
        _lib.check(L.h2g_shard_load_q(self._plan, C.c_void_p(q_own.data_ptr()),
                                      C.c_void_p(stream)), "h2g_shard_load_q", L=L)
        if self.nranks > 1:
            hm = max(1, self.info["max_halo_slots"])
            if getattr(self, "_hsend", None) is None:
                dev = f"cuda:{self.device}"
                self._hsend = torch.zeros(hm, dtype=torch.float64, device=dev)
                self._hrecv = torch.zeros(hm * self.nranks, dtype=torch.float64, device=dev)
            _lib.check(L.h2g_halo_pack(self._plan, C.c_void_p(self._hsend.data_ptr()),
                                       C.c_void_p(stream)), "h2g_halo_pack", L=L)
            dist.all_gather_into_tensor(self._hrecv, self._hsend, group=self.group)
            _lib.check(L.h2g_halo_unpack(self._plan, C.c_void_p(self._hrecv.data_ptr()),
                                         C.c_void_p(stream)), "h2g_halo_unpack", L=L)
            _lib.check(L.h2g_shard_part0(self._plan, C.c_void_p(stream)), "h2g_shard_part0", L=L)
            send, recv = self._buffers(torch)
            self.pack(send, stream)
            self._all_gather_overlapped(dist, recv, send, stream)
            self.unpack(recv, stream)
        else:
            raise ValueError("matvec_distributed needs a sharded plan (nranks > 1)")
        _lib.check(L.h2g_shard_store_phi(self._plan, C.c_void_p(phi_own.data_ptr()),
                                         C.c_void_p(stream)), "h2g_shard_store_phi", L=L)
        return phi_own

    def matvec(self, q, gather_full: bool = False):
        """phi = K~ q on this rank's rows (torch CUDA tensor q, replicated)."""
        import torch
        import torch.distributed as dist
        if q.shape[0] != self.N:
            raise ValueError("vector length mismatch")
        q = q.to(torch.float64).contiguous()
        stream = torch.cuda.current_stream(q.device).cuda_stream
        phi = torch.zeros_like(q)
        send, recv = self._buffers(torch)
        self.begin(q, stream)
        if self.nranks > 1:
            self.pack(send, stream)
            self._all_gather_overlapped(dist, recv, send, stream)
            self.unpack(recv, stream)
        self.end(phi, stream)
        if gather_full and self.nranks > 1:
            dist.all_reduce(phi, group=self.group)  # disjoint rows: exact
        return phi


# ------------------------------------------------------------ CPU emulation
def schedule_view(op: PackedOperator, rank: int = 0, nranks: int = 1, recompute: str = "") -> dict:
    """Rank's host schedule (include/h2g.h h2g_schedule_build) as numpy arrays;
    ``recompute`` as for GpuHierRep (blocks evaluated even where stored)."""
    L = _lib.load()
    desc, keep = _desc_from_packed(op, recompute)
    h = C.c_void_p()
    _lib.check(L.h2g_schedule_build(C.byref(desc), int(rank), int(nranks), C.byref(h)),
               "h2g_schedule_build")
    out = {}
    try:
        for name, cols in (("tasks", 5), ("terms", 6), ("phases", 4), ("pack", 3),
                           ("unpack", 3), ("meta", 1), ("blob", 1), ("recs", 4), ("halo", 3)):
            ptr, n, is_f64 = C.c_void_p(), C.c_int64(), C.c_int32()
            _lib.check(L.h2g_schedule_get(h, name.encode(), C.byref(ptr), C.byref(n),
                                          C.byref(is_f64)))
            dt = np.float64 if is_f64.value else np.int64
            if n.value:
                buf = (C.c_char * (n.value * 8)).from_address(ptr.value)
                a = np.frombuffer(buf, dtype=dt, count=n.value).copy()
            else:
                a = np.zeros(0, dt)
            out[name] = a.reshape(-1, cols) if cols > 1 else a
    finally:
        L.h2g_schedule_free(h)
    del keep
    m = out["meta"]
    out.update(n_slots=int(m[0]), q_tree=int(m[1]), phi_tree=int(m[2]), ones_off=int(m[3]),
               n_ones=int(m[4]), row_begin=int(m[5]), row_end=int(m[6]), send_slots=int(m[7]),
               max_send_slots=int(m[8]), level=int(m[9]))
    return out
