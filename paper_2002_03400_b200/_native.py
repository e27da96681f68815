"""Loader for the in-tree CUDA library (``_native/libbfly_b200.so``).

There is no CPU fallback: if the library is missing the import of the
product API raises, and every compute entry point needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BFLY_LIB: an alternative in-tree build of the same library (A/B experiments, tools/)
LIB_PATH = os.environ.get("BFLY_LIB") or os.path.join(_HERE, "_native", "libbfly_b200.so")

_lib = None


class BflyError(RuntimeError):
    """Base of the reference's error hierarchy (core.hpp:43-60)."""

    code = -1


class PreconditionError(BflyError):
    code = 1


class DimensionError(BflyError):
    code = 2


class SequencingError(BflyError):
    code = 3


class FormatError(BflyError):
    code = 4


class ConditioningError(BflyError):
    code = 5


class CudaError(BflyError):
    code = 6


class NcclError(BflyError):
    code = 7


_ERRORS = {c.code: c for c in (PreconditionError, DimensionError, SequencingError, FormatError,
                                ConditioningError, CudaError, NcclError)}


class Cfg(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double), ("oversampling", C.c_int64), ("rank_guess", C.c_int64),
        ("levels", C.c_int32), ("center", C.c_int32), ("seed", C.c_uint64), ("hard_cap", C.c_int64),
        ("threads", C.c_int32), ("literal_transpose_core", C.c_int32), ("max_batch_probes", C.c_int64),
        ("virtual_ranks", C.c_int32), ("reserved_", C.c_int32),
    ]


class Phase(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("forward_columns", C.c_int64), ("transpose_columns", C.c_int64),
                ("seconds", C.c_double), ("rounds", C.c_int32), ("probe_width", C.c_int64),
                ("rank_margin", C.c_double)]


class Log(C.Structure):
    _fields_ = [("nphases", C.c_int32), ("phases", Phase * 64), ("peak_probe_bytes", C.c_uint64),
                ("peak_concurrent_probes", C.c_int64), ("rank_capped", C.c_int32), ("total_seconds", C.c_double),
                ("flops", C.c_double), ("kernel_evals", C.c_double), ("products_recomputed", C.c_int32)]


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                       C.c_void_p)
APPLY_RANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                             C.c_int64, C.c_int64, C.c_void_p)


# bfly_host_comm (include/bfly_b200.h): host-staged collectives supplied by the caller
HC_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)
HC_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int)
HC_SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                          C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                          C.POINTER(C.c_int64))


class HostCommFns(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", HC_ALLGATHER), ("allreduce", HC_ALLREDUCE),
                ("sendrecv", HC_SENDRECV)]


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    p, i64, u64, i32, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double
    pp = C.POINTER(C.c_void_p)
    sig = {
        "bfly_last_error": (C.c_char_p, []),
        "bfly_version": (C.c_char_p, []),
        "bfly_ctx_create": (i32, [i32, pp]),
        "bfly_ctx_destroy": (i32, [p]),
        "bfly_ctx_launches": (i64, [p]),
        "bfly_ctx_synchronize": (i32, [p]),
        "bfly_ctx_stream": (p, [p]),
        "bfly_ctx_profile": (i32, [p, i32]),
        "bfly_ctx_profile_report": (i64, [p, C.c_char_p, i64]),
        "bfly_comm_unique_id": (i32, [p]),
        "bfly_ctx_set_comm": (i32, [p, i32, i32, p]),
        "bfly_ctx_set_host_comm": (i32, [p, i32, i32, C.POINTER(HostCommFns)]),
        "bfly_ctx_comm_info": (i32, [p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "bfly_tree_build": (i32, [i32, i64, p, i32, pp]),
        "bfly_tree_from_table": (i32, [i64, i32, p, p, pp]),
        "bfly_tree_info": (i32, [p, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
        "bfly_tree_table": (i32, [p, p, p]),
        "bfly_tree_destroy": (None, [p]),
        "bfly_depth_for": (i32, [i64, i64]),
        "bfly_points_uniform": (None, [i64, u64, u64, dbl, dbl, p]),
        "bfly_points_plate": (None, [i64, dbl, p]),
        "bfly_points_half_circle": (None, [i64, i32, p]),
        "bfly_op_kernel": (i32, [p, i32, i64, i64, p, p, dbl, i32, pp]),
        "bfly_op_compose": (i32, [p, p, p, pp]),
        "bfly_op_dense": (i32, [p, i64, i64, p, i32, pp]),
        "bfly_op_butterfly": (i32, [p, p, pp]),
        "bfly_op_callback": (i32, [p, i64, i64, i32, APPLY_FN, p, pp]),
        "bfly_op_callback_ranged": (i32, [p, i64, i64, i32, APPLY_RANGE_FN, p, pp]),
        "bfly_op_info": (i32, [p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "bfly_op_apply": (i32, [p, i32, p, i64, p, i64, i64, i32]),
        "bfly_op_counters": (i32, [p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "bfly_op_reset_counters": (i32, [p]),
        "bfly_op_destroy": (None, [p]),
        "bfly_cfg_default": (None, [C.POINTER(Cfg)]),
        "bfly_factorize": (i32, [p, p, p, p, C.POINTER(Cfg), pp, C.POINTER(Log)]),
        "bfly_factorizer_create": (i32, [p, p, p, p, C.POINTER(Cfg), pp]),
        "bfly_factorizer_leaf_row_bases": (i32, [p]),
        "bfly_factorizer_leaf_col_bases": (i32, [p]),
        "bfly_factorizer_transfer_level_w": (i32, [p, i32]),
        "bfly_factorizer_transfer_level_r": (i32, [p, i32]),
        "bfly_factorizer_complete": (i32, [p]),
        "bfly_factorizer_take": (i32, [p, pp, C.POINTER(Log)]),
        "bfly_factorizer_destroy": (None, [p]),
        "bfly_estimate_error": (i32, [p, p, i64, u64, C.POINTER(C.c_double)]),
        "bfly_residuals": (i32, [p, p, p, p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "bfly_apply": (i32, [p, i32, p, i64, p, i64, i64, i32]),
        "bfly_apply_layout": (i32, [p, i32, i32, i64, p, i64, p, i64, i64, i32, C.POINTER(C.c_double)]),
        "bfly_comm_cost": (i32, [i32, i32, i64, i64, C.POINTER(C.c_double)]),
        "bfly_layout_owners": (i64, [i32, i32, i32, i64, p]),
        "bfly_bf_info": (i32, [p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int)]),
        "bfly_rank_profile": (i64, [p, p]),
        "bfly_serialize": (i64, [p, p]),
        "bfly_deserialize": (i32, [p, p, i64, i32, pp]),
        "bfly_synth_butterfly": (i32, [p, i32, i64, i64, u64, i32, dbl, pp]),
        "bfly_bf_convert": (i32, [p, i32, pp]),
        "bfly_bf_destroy": (None, [p]),
        "bfly_gaussian": (i32, [p, i64, i64, u64, i32, p]),
        "bfly_seed_mix": (u64, [u64, i32, p]),
        "bfly_cpqr_truncate": (i32, [p, i64, i64, p, dbl, p, C.POINTER(C.c_int64)]),
        "bfly_pinv": (i32, [p, i64, i64, p, dbl, p]),
        "bfly_vrank_times": (i64, [p, i64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(code):
    if code != 0:
        msg = lib().bfly_last_error().decode(errors="replace")
        raise _ERRORS.get(code, BflyError)(msg)
