"""ctypes binding of libpbq.so (the C ABI declared in include/pbq.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2103_07245_b200.build``).  There is no fallback: if the
library is missing or no CUDA device is present every entry point raises.
"""
import ctypes
import os
import threading

from . import exceptions as _exc

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpbq.so")

PBQ_OK = 0
PBQ_ERR_PARAM = 1
PBQ_ERR_DIM = 2
PBQ_ERR_NONFINITE = 3
PBQ_ERR_CUDA = 4
PBQ_ERR_NCCL = 5
PBQ_ERR_OOM = 6
PBQ_ERR_UNSUPPORTED = 7

# every symbol include/pbq.h declares (checked by tests/test_boundary.py)
EXPORTED = (
    "pbq_ctx_create",
    "pbq_ctx_destroy",
    "pbq_last_error",
    "pbq_ctx_sm_count",
    "pbq_ctx_launch_count",
    "pbq_gemm_tn",
    "pbq_gemm_nn",
    "pbq_gemm_workspace_bytes",
    "pbq_householder_qr",
    "pbq_qr_workspace_bytes",
    "pbq_gaussian",
    "pbq_gaussian_workspace_bytes",
    "pbq_pbp_qlp_workspace_bytes",
    "pbq_pbp_qlp",
    "pbq_transpose",
    "pbq_second_stage",
    "pbq_second_stage_workspace_bytes",
    "pbq_gemm_tn_scatter",
    "pbq_xchg_reduce",
    "pbq_xchg_wait",
    "pbq_xchg_expected_tiles",
    "pbq_p2p_push",
    "pbq_p2p_sum",
    "pbq_p2p_wait",
    "pbq_debug_qr_hooks",
    "pbq_profile_begin",
    "pbq_profile_end",
    "pbq_set_qr_method",
    "pbq_debug_cholqr_stats",
    "pbq_residual_fro",
    "pbq_residual_workspace_bytes",
    "pbq_cpqr_pivots",
    "pbq_cpqr_workspace_bytes",
    "pbq_gather_columns",
    "pbq_cholqr2_dist",
    "pbq_cholqr2_dist_workspace_bytes",
    "pbq_set_p2p_timeout_ms",
    "pbq_jacobi_svd",
    "pbq_jacobi_svd_workspace_bytes",
    "pbq_clear_error",
    "pbq_orth_basis",
    "pbq_set_basis_orth",
)

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_p = ctypes.c_void_p
c_i32 = ctypes.c_int32
c_sz = ctypes.c_size_t
c_dbl = ctypes.c_double


class PbqProblem(ctypes.Structure):
    _fields_ = [
        ("n1", c_i64), ("n2", c_i64), ("d", c_i64), ("q", c_i64),
        ("a", c_p), ("lda", c_i64),
        ("phi", c_p), ("ldphi", c_i64),
        ("seed_lo", c_u64), ("seed_hi", c_u64),
        ("reorthonormalize", c_i32), ("check_finite", c_i32),
        ("c_init", c_p), ("ldc_init", c_i64),
        ("seed_dev", c_p),
    ]


class PbqOutputs(ctypes.Structure):
    _fields_ = [
        ("q", c_p), ("ldq", c_i64),
        ("l", c_p), ("ldl", c_i64),
        ("p", c_p), ("ldp", c_i64),
        ("r", c_p), ("ldr", c_i64),
        ("phi", c_p), ("ldphi", c_i64),
        ("rank_flags", c_p),
        ("nonfinite", c_p),
    ]


_SIGS = {
    "pbq_ctx_create": ([ctypes.c_int, ctypes.POINTER(c_p)], ctypes.c_int),
    "pbq_ctx_destroy": ([c_p], ctypes.c_int),
    "pbq_last_error": ([c_p], ctypes.c_char_p),
    "pbq_ctx_sm_count": ([c_p], ctypes.c_int),
    "pbq_ctx_launch_count": ([c_p], c_i64),
    "pbq_gemm_tn": ([c_p, c_i64, c_i64, c_i64, c_dbl, c_p, c_i64, c_p, c_i64, c_dbl, c_p, c_i64, c_p, c_p, c_sz, c_p],
                    ctypes.c_int),
    "pbq_gemm_nn": ([c_p, c_i64, c_i64, c_i64, c_dbl, c_p, c_i64, c_p, c_i64, c_dbl, c_p, c_i64, c_p, c_p, c_sz, c_p],
                    ctypes.c_int),
    "pbq_gemm_workspace_bytes": ([c_p, c_i64, c_i64, c_i64, ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_householder_qr": ([c_p, c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_i32, c_p, c_p, c_sz, c_p], ctypes.c_int),
    "pbq_qr_workspace_bytes": ([c_p, c_i64, c_i64, ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_gaussian": ([c_p, c_i64, c_i64, c_i64, c_u64, c_u64, c_p, c_i64, c_p, c_p, c_sz, c_p], ctypes.c_int),
    "pbq_gaussian_workspace_bytes": ([c_p, c_i64, c_i64, c_i64, ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_pbp_qlp_workspace_bytes": ([c_p, ctypes.POINTER(PbqProblem), ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_pbp_qlp": ([c_p, ctypes.POINTER(PbqProblem), ctypes.POINTER(PbqOutputs), c_p, c_sz, c_p], ctypes.c_int),
    "pbq_transpose": ([c_p, c_i64, c_p, c_i64, c_p, c_i64, c_i32, c_p], ctypes.c_int),
    "pbq_second_stage": ([c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_sz, c_p], ctypes.c_int),
    "pbq_second_stage_workspace_bytes": ([c_p, c_i64, ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_gemm_tn_scatter": ([c_p, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_p, c_i32, c_i32, c_i64, c_i64, c_p,
                             c_p, c_sz, c_p], ctypes.c_int),
    "pbq_xchg_reduce": ([c_p, c_i32, c_i32, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, ctypes.c_uint32, c_p, c_p],
                        ctypes.c_int),
    "pbq_xchg_wait": ([c_p, c_p, ctypes.c_uint32, c_p], ctypes.c_int),
    "pbq_xchg_expected_tiles": ([c_i64, c_i64, c_i64, c_i32, c_i32, ctypes.POINTER(ctypes.c_uint32)], ctypes.c_int),
    "pbq_p2p_push": ([c_p, c_p, c_i64, c_p, c_i64, c_i32, c_i32, c_p, c_p], ctypes.c_int),
    "pbq_p2p_sum": ([c_p, c_p, c_i64, c_i32, c_i64, c_p, c_p, ctypes.c_uint32, c_p, c_p], ctypes.c_int),
    "pbq_p2p_wait": ([c_p, c_p, ctypes.c_uint32, c_p, c_p], ctypes.c_int),
    "pbq_set_p2p_timeout_ms": ([c_p, c_i64], ctypes.c_int),
    "pbq_clear_error": ([c_p], ctypes.c_int),
    "pbq_jacobi_svd": ([c_p, c_i64, c_i64, c_p, c_i64, c_i32, c_p, c_p, c_i64, c_p, c_i64, c_p, c_p, c_sz, c_p],
                       ctypes.c_int),
    "pbq_jacobi_svd_workspace_bytes": ([c_p, c_i64, c_i64, c_i32, ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_debug_qr_hooks": ([c_p, c_p, c_p, c_p], ctypes.c_int),
    "pbq_profile_begin": ([c_p, c_i32], ctypes.c_int),
    "pbq_profile_end": ([c_p, ctypes.POINTER(c_dbl), ctypes.POINTER(c_i32)], ctypes.c_int),
    "pbq_set_qr_method": ([c_p, c_i32], ctypes.c_int),
    "pbq_set_basis_orth": ([c_p, c_i32], ctypes.c_int),
    "pbq_orth_basis": ([c_p, c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_p, c_sz, c_p], ctypes.c_int),
    "pbq_residual_fro": ([c_p, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_p, c_sz, c_p],
                         ctypes.c_int),
    "pbq_residual_workspace_bytes": ([c_p, c_i64, c_i64, c_i64, ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_debug_cholqr_stats": ([c_p, c_p], ctypes.c_int),
    "pbq_cpqr_pivots": ([c_p, c_i64, c_i64, c_p, c_i64, c_p, c_p, c_sz, c_p], ctypes.c_int),
    "pbq_cpqr_workspace_bytes": ([c_p, c_i64, c_i64, ctypes.POINTER(c_sz)], ctypes.c_int),
    "pbq_gather_columns": ([c_p, c_i64, c_i64, c_p, c_i64, c_p, c_p, c_i64, c_p], ctypes.c_int),
    "pbq_cholqr2_dist": ([c_p, c_i32, c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_p, c_sz, c_p],
                         ctypes.c_int),
    "pbq_cholqr2_dist_workspace_bytes": ([c_p, c_i64, c_i64, ctypes.POINTER(c_sz), ctypes.POINTER(c_i64)],
                                         ctypes.c_int),
}

_lib = None
_lib_lock = threading.Lock()


def load():
    """Load libpbq.so (raises if it has not been built)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise _exc.DeviceError(
                    f"{LIB_PATH} is missing: build the CUDA library first "
                    "(python -c 'import __graft_entry__ as g; g.build()')"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (argtypes, restype) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = restype
            _lib = lib
    return _lib


def raise_status(status, ctx, what):
    """Map a pbq_status to the reference's exception classes."""
    if status == PBQ_OK:
        return
    msg = load().pbq_last_error(ctx)
    msg = msg.decode() if msg else ""
    text = f"{what}: {msg}" if msg else what
    if status == PBQ_ERR_PARAM:
        raise _exc.ParameterError(text)
    if status == PBQ_ERR_DIM:
        raise _exc.DimensionError(text)
    if status == PBQ_ERR_NONFINITE:
        raise _exc.MatrixInputError(text)
    if status == PBQ_ERR_OOM:
        raise MemoryError(text)
    raise _exc.DeviceError(f"{text} (status {status})")
