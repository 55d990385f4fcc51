"""Exception and warning types of the PbP-QLP path.

Same hierarchy and meaning as the reference's
(/root/reference/pkg/src/pbpqlp/exceptions.py:8-57) so that callers catching
``ValueError``/``ParameterError`` keep working when this package is swapped in.
Only the types the PbP-QLP path raises are defined here.
"""


class ParameterError(ValueError):
    """An argument is outside its documented range (exceptions.py:8)."""


class DimensionError(ParameterError):
    """A matrix dimension is zero or negative (exceptions.py:12)."""


class MatrixInputError(ValueError):
    """A matrix argument is malformed: wrong rank, non-numeric, or non-finite
    (exceptions.py:16)."""


class RankDeficiencyWarning(UserWarning):
    """An orthonormalization met numerically dependent columns; the basis is
    still returned (exceptions.py:56-57)."""


class ConvergenceError(RuntimeError):
    """An iterative kernel failed to converge; ``estimate`` carries the best
    value reached (exceptions.py:37-44)."""

    def __init__(self, message, estimate=None):
        super().__init__(message)
        self.estimate = estimate


class DeviceError(RuntimeError):
    """The CUDA library reported a failure (launch, memory, unsupported shape)."""
