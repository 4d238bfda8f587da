"""ctypes binding of the C ABI in include/h2g.h (libh2g.so).

The library is built in-tree (paper_2309_14085_b200/build.py).  Loading
fails loudly if it is missing: there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import os

LIBDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")

H2G_ABI_VERSION = 3
H2G_RECOMPUTE_NEAR = 1
H2G_RECOMPUTE_M2L = 2
H2G_KERNELS = {"log2d": 0, "lap3d": 1, "gaussian": 2}
H2G_OK = 0
H2G_ERR_LENGTH_MISMATCH = 1

P_I32 = C.POINTER(C.c_int32)
P_I64 = C.POINTER(C.c_int64)
P_F64 = C.POINTER(C.c_double)


class ChannelDesc(C.Structure):
    _fields_ = [("r_in", P_I32), ("r_out", P_I32), ("p2m_off", P_I64), ("l2p_off", P_I64),
                ("m2m_off", P_I64), ("l2l_off", P_I64), ("m2l_rowptr", P_I64),
                ("m2l_src", P_I32), ("m2l_off", P_I64), ("piv_in_ptr", P_I64),
                ("piv_in", P_I64), ("piv_out_ptr", P_I64), ("piv_out", P_I64)]


class ExportDesc(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("dim", C.c_int32), ("kappa", C.c_int32),
                ("n_channels", C.c_int32), ("n_points", C.c_int64), ("n_clusters", C.c_int64),
                ("mem_scalars", C.c_int64), ("perm", P_I64), ("level_offset", P_I64),
                ("cl_start", P_I64), ("cl_end", P_I64), ("channels", ChannelDesc * 2),
                ("blr_rowptr", P_I64), ("blr_src", P_I32), ("blr_rank", P_I32),
                ("blr_u_off", P_I64), ("blr_v_off", P_I64), ("near_rowptr", P_I64),
                ("near_src", P_I32), ("near_off", P_I64), ("blob_len", C.c_int64),
                ("blob", P_F64), ("points_tree", P_F64), ("kernel_type", C.c_int32),
                ("has_diag", C.c_int32), ("zero_value", C.c_double), ("diag", C.c_double),
                ("shift", C.c_double), ("sigma", C.c_double), ("recompute", C.c_int32),
                ("pad0", C.c_int32), ("m2l_recompute_share", C.c_double)]


class PlanStats(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("mem_scalars", C.c_int64), ("alg_bytes", C.c_int64),
                ("blob_bytes", C.c_int64), ("workspace_bytes", C.c_int64),
                ("n_phases", C.c_int32), ("n_launches", C.c_int32), ("n_tasks", C.c_int64),
                ("n_terms", C.c_int64), ("device", C.c_int32), ("graph", C.c_int32)]


class ShardInfo(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("level", C.c_int32),
                ("pad", C.c_int32), ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("send_slots", C.c_int64), ("max_send_slots", C.c_int64),
                ("blob_bytes", C.c_int64), ("halo_slots", C.c_int64),
                ("max_halo_slots", C.c_int64)]


# every symbol include/h2g.h declares (checked by tests/test_abi.py)
H2G_SYMBOLS = ("h2g_plan_create", "h2g_plan_destroy", "h2g_plan_get_stats", "h2g_matvec",
               "h2g_matvec_host", "h2g_profile_phases", "h2g_profile_phases_batched", "h2g_schedule_info",
               "h2g_launches_per_matvec",
               "h2g_error_string", "h2g_last_error_detail", "h2g_abi_version",
               "h2g_plan_create_sharded", "h2g_shard_get_info", "h2g_matvec_begin",
               "h2g_shard_pack", "h2g_shard_unpack", "h2g_matvec_end",
               "h2g_schedule_build", "h2g_schedule_get", "h2g_schedule_free",
               "h2g_shard_load_q", "h2g_halo_pack", "h2g_halo_unpack", "h2g_shard_part0",
               "h2g_shard_store_phi", "h2g_shard_overlap")

_LIB = None


def lib_path() -> str:
    # H2G_LIB_PATH: load an alternative build (diagnostic builds in experiments)
    return os.environ.get("H2G_LIB_PATH") or os.path.join(LIBDIR, "libh2g.so")


def load(path: str = None) -> C.CDLL:
    """Load libh2g.so (raises if it was not built).  ``path`` loads a specific
    build uncached (side-by-side variants in experiments)."""
    global _LIB
    if path is None and _LIB is not None:
        return _LIB
    explicit = path is not None
    path = path or lib_path()
    if not os.path.exists(path):
        raise RuntimeError(
            f"native library {path} is missing; build it with "
            "`python -m paper_2309_14085_b200.build` (no CPU fallback exists)")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.h2g_plan_create.argtypes = [C.POINTER(ExportDesc), C.c_int, C.POINTER(vp)]
    L.h2g_plan_destroy.argtypes = [vp]
    L.h2g_plan_get_stats.argtypes = [vp, C.POINTER(PlanStats)]
    L.h2g_matvec.argtypes = [vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, vp]
    L.h2g_matvec_host.argtypes = [vp, P_F64, P_F64, C.c_int64, C.c_int64, C.c_int64]
    L.h2g_profile_phases.argtypes = [vp, vp, vp, C.c_int, P_F64, P_I64,
                                     C.POINTER(C.c_char_p), C.c_int, C.POINTER(C.c_int)]
    L.h2g_profile_phases_batched.argtypes = [vp, C.c_int, C.c_int, P_F64, P_I64,
                                             C.POINTER(C.c_char_p), C.c_int, C.POINTER(C.c_int)]
    L.h2g_launches_per_matvec.argtypes = [vp, C.c_int64]
    L.h2g_schedule_info.argtypes = [C.POINTER(ExportDesc), C.c_int, C.c_char_p, C.c_int64]
    L.h2g_plan_create_sharded.argtypes = [C.POINTER(ExportDesc), C.c_int, C.c_int, C.c_int,
                                          C.POINTER(vp)]
    L.h2g_shard_get_info.argtypes = [vp, C.POINTER(ShardInfo)]
    L.h2g_matvec_begin.argtypes = [vp, vp, C.c_int64, vp]
    L.h2g_shard_pack.argtypes = [vp, vp, vp]
    L.h2g_shard_unpack.argtypes = [vp, vp, vp]
    L.h2g_matvec_end.argtypes = [vp, vp, C.c_int64, vp]
    for name in ("h2g_shard_load_q", "h2g_halo_pack", "h2g_halo_unpack", "h2g_shard_store_phi"):
        getattr(L, name).argtypes = [vp, vp, vp]
    L.h2g_shard_part0.argtypes = [vp, vp]
    L.h2g_shard_overlap.argtypes = [vp, vp]
    L.h2g_schedule_build.argtypes = [C.POINTER(ExportDesc), C.c_int, C.c_int, C.POINTER(vp)]
    L.h2g_schedule_get.argtypes = [vp, C.c_char_p, C.POINTER(vp), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int32)]
    L.h2g_schedule_free.argtypes = [vp]
    L.h2g_schedule_free.restype = None
    L.h2g_error_string.argtypes = [C.c_int]
    L.h2g_error_string.restype = C.c_char_p
    L.h2g_last_error_detail.restype = C.c_char_p
    if L.h2g_abi_version() != H2G_ABI_VERSION:
        raise RuntimeError("libh2g.so ABI version mismatch; rebuild it")
    if not explicit:
        _LIB = L
    return L


def check(rc: int, what: str = "h2g", L=None):
    if rc == H2G_OK:
        return
    L = L or load()
    msg = L.h2g_error_string(rc).decode()
    detail = L.h2g_last_error_detail().decode()
    if rc == H2G_ERR_LENGTH_MISMATCH:
        raise ValueError("vector length mismatch")
    raise RuntimeError(f"{what}: {msg}" + (f" ({detail})" if detail else ""))
