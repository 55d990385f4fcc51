"""B200-native PbP-QLP (projection-based partial QLP, arXiv:2103.07245).

Drop-in for the reference package's PbP-QLP path (``pbpqlp.pbp_qlp``,
/root/reference/pkg/src/pbpqlp/algorithms.py:209-260): same entry point,
arguments, errors, warnings and result fields; every FLOP runs in
hand-written sm_100a CUDA behind the C ABI in include/pbq.h.
"""
from .algorithms import (PbpQlpPlan, QlpFactors, SketchRecord, clear_plan_cache, pbp_qlp, pbp_qlp_bytes,
                         pbp_qlp_flops, reconstruction_error, residual_norms)
from .exceptions import (ConvergenceError, DeviceError, DimensionError, MatrixInputError, ParameterError,
                         RankDeficiencyWarning)
from .multigpu import MultiGpuPool, pbp_qlp_multi_gpu
from .linalg import QrFactors, column_pivoted_qr, gaussian_matrix, householder_qr, orth
from .rsvd import RsvdFactors, r_svd
from .utv import UtvFactors, cor_utv

__version__ = "0.1.0"

__all__ = [
    "ConvergenceError",
    "DeviceError",
    "DimensionError",
    "MatrixInputError",
    "MultiGpuPool",
    "ParameterError",
    "PbpQlpPlan",
    "QlpFactors",
    "QrFactors",
    "RankDeficiencyWarning",
    "RsvdFactors",
    "SketchRecord",
    "UtvFactors",
    "clear_plan_cache",
    "column_pivoted_qr",
    "cor_utv",
    "gaussian_matrix",
    "householder_qr",
    "orth",
    "pbp_qlp",
    "pbp_qlp_bytes",
    "pbp_qlp_flops",
    "pbp_qlp_multi_gpu",
    "r_svd",
    "reconstruction_error",
    "residual_norms",
    "__version__",
]
