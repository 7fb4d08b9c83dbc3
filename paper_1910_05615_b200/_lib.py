"""ctypes binding of libpaper_1910_05615_b200.so (include/rtdetmcd.h).

Argument marshalling only: every step of the method runs in the library's
CUDA kernels.  Importing this module never falls back to anything: if the
shared library is missing, `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpaper_1910_05615_b200.so")

RTD_STATUS = {
    0: "RTD_OK", 1: "RTD_E_INVALID_ARG", 2: "RTD_E_NONFINITE", 3: "RTD_E_DEGENERATE_COLUMN",
    4: "RTD_E_BOTH_STARTS_FAILED", 5: "RTD_E_TOO_FEW_VALID_BLOCKS", 6: "RTD_E_NOT_PD", 7: "RTD_E_CUDA",
    8: "RTD_E_OOM", 9: "RTD_E_INTERNAL", 10: "RTD_E_NCCL",
}

EXPORTS = [
    "rtdetmcd_opts_default", "rtdetmcd_create", "rtdetmcd_destroy", "rtdetmcd_last_error",
    "rtdetmcd_set_workspace", "rtdetmcd_fit_workspace_size", "rtdetmcd_fit", "rtdetmcd_fit_warm", "rtdetmcd_fit_batches", "rtdetmcd_flag",
    "rtdetmcd_unimcd", "rtdetmcd_initial", "rtdetmcd_refine", "rtdetmcd_csteps",
    "rtdetmcd_chi2_quantile", "rtdetmcd_consistency_factor", "rtdetmcd_choose_q", "rtdetmcd_partition_perm",
    "rtdetmcd_set_profiling", "rtdetmcd_prof_count", "rtdetmcd_prof_entry", "rtdetmcd_counters",
    "rtdetmcd_moment_doubles", "rtdetmcd_columns", "rtdetmcd_blocks_fit", "rtdetmcd_aggregate",
    "rtdetmcd_blocks_reweight", "rtdetmcd_pool_reweight",
    "rtdetmcd_nccl_unique_id", "rtdetmcd_create_dist", "rtdetmcd_create_transport", "rtdetmcd_shard_layout",
    "rtdetmcd_fit_sharded", "rtdetmcd_ctx_comm",
]

# rtdetmcd_transport callbacks (host buffers)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                           C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t))


class Transport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", ALLGATHER_FN), ("alltoallv", ALLTOALLV_FN)]


class Opts(C.Structure):
    _fields_ = [
        ("h", C.c_int64), ("alpha", C.c_double), ("shards", C.c_int32), ("shard_cap", C.c_int32),
        ("omega", C.c_int64), ("kappa_max", C.c_double), ("quantile", C.c_double), ("max_csteps", C.c_int32),
        ("refresh_every", C.c_int32), ("seed", C.c_uint64), ("partition", C.c_int32), ("log_transform", C.c_int32),
        ("distance", C.c_int32), ("consistency", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("loc", C.c_void_p), ("scale", C.c_void_p), ("mu_raw", C.c_void_p), ("sigma_raw", C.c_void_p),
        ("mu_rew", C.c_void_p), ("sigma_rew", C.c_void_p),
        ("logdet_raw", C.c_double), ("cutoff2", C.c_double), ("h", C.c_int64), ("h_block", C.c_int64),
        ("m", C.c_int64), ("q_used", C.c_int32), ("warnings", C.c_int32), ("n_valid_blocks", C.c_int32),
        ("n_kept_blocks", C.c_int32), ("n_weighted", C.c_int64),
        ("block_chosen", C.c_void_p), ("start_steps", C.c_void_p), ("start_status", C.c_void_p),
        ("start_logdet", C.c_void_p),
        ("flags", C.c_void_p), ("rd2", C.c_void_p), ("weights", C.c_void_p), ("hsubset", C.c_void_p),
    ]


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    L.rtdetmcd_opts_default.argtypes = [C.POINTER(Opts)]
    L.rtdetmcd_opts_default.restype = None
    L.rtdetmcd_create.argtypes = [C.POINTER(vp), C.c_int, vp]
    L.rtdetmcd_destroy.argtypes = [vp]
    L.rtdetmcd_destroy.restype = None
    L.rtdetmcd_last_error.argtypes = [vp]
    L.rtdetmcd_last_error.restype = C.c_char_p
    L.rtdetmcd_set_workspace.argtypes = [vp, vp, C.c_size_t]
    L.rtdetmcd_fit_workspace_size.argtypes = [i64, i32, C.POINTER(Opts)]
    L.rtdetmcd_fit_workspace_size.restype = C.c_size_t
    L.rtdetmcd_fit.argtypes = [vp, vp, i64, i32, C.POINTER(Opts), C.POINTER(Result)]
    L.rtdetmcd_fit_warm.argtypes = [vp, vp, i64, i32, C.POINTER(Opts), vp, vp, C.POINTER(Result)]
    L.rtdetmcd_fit_batches.argtypes = [vp, C.POINTER(C.c_void_p), i32, i64, i32, C.POINTER(Opts), C.POINTER(Result)]
    L.rtdetmcd_flag.argtypes = [vp, vp, i64, i32, vp, vp, f64, i32, vp, vp]
    L.rtdetmcd_unimcd.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp, vp]
    L.rtdetmcd_initial.argtypes = [vp, vp, i64, i32, vp, vp, vp]
    L.rtdetmcd_refine.argtypes = [vp, vp, i64, i32, vp, f64, vp, vp, vp, vp]
    L.rtdetmcd_csteps.argtypes = [vp, vp, i64, i32, i64, vp, vp, f64, i32, i32, vp, vp, vp, vp, vp, vp, vp]
    L.rtdetmcd_chi2_quantile.argtypes = [f64, i32]
    L.rtdetmcd_chi2_quantile.restype = f64
    L.rtdetmcd_consistency_factor.argtypes = [f64, i32]
    L.rtdetmcd_consistency_factor.restype = f64
    L.rtdetmcd_choose_q.argtypes = [i64, i32, i64, i32]
    L.rtdetmcd_choose_q.restype = i32
    L.rtdetmcd_partition_perm.argtypes = [vp, i64, u64, vp]
    L.rtdetmcd_set_profiling.argtypes = [vp, i32]
    L.rtdetmcd_moment_doubles.argtypes = [i32]
    L.rtdetmcd_moment_doubles.restype = i32
    L.rtdetmcd_columns.argtypes = [vp, vp, i64, i32, i32, vp]
    L.rtdetmcd_blocks_fit.argtypes = [vp, vp, i64, i32, vp, vp, i32, i32, i64, C.POINTER(Opts), vp]
    L.rtdetmcd_aggregate.argtypes = [vp, i32, i32, i64, vp, vp, vp, vp]
    L.rtdetmcd_blocks_reweight.argtypes = [vp, f64, vp, vp]
    L.rtdetmcd_pool_reweight.argtypes = [vp, i32, vp, f64, vp, vp, vp, vp, vp]
    L.rtdetmcd_nccl_unique_id.argtypes = [vp]
    L.rtdetmcd_create_dist.argtypes = [C.POINTER(vp), C.c_int, vp, vp, C.c_int, C.c_int]
    L.rtdetmcd_create_transport.argtypes = [C.POINTER(vp), C.c_int, vp, C.POINTER(Transport), C.c_int, C.c_int]
    L.rtdetmcd_shard_layout.argtypes = [i64, i32, i32, i32, vp, vp, vp, vp]
    L.rtdetmcd_fit_sharded.argtypes = [vp, vp, i64, i64, i32, C.POINTER(Opts), C.POINTER(Result)]
    L.rtdetmcd_ctx_comm.argtypes = [vp, vp, vp, C.POINTER(C.c_char_p)]
    L.rtdetmcd_counters.argtypes = [vp, vp]
    L.rtdetmcd_counters.restype = None
    L.rtdetmcd_prof_count.argtypes = [vp]
    L.rtdetmcd_prof_count.restype = i32
    L.rtdetmcd_prof_entry.argtypes = [vp, i32, C.c_char_p, C.c_size_t, vp, vp, vp, vp, vp]
    for name in EXPORTS:  # every declared symbol must resolve
        getattr(L, name)
    _LIB = L
    return L
