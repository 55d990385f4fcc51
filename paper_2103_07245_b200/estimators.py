"""scikit-learn transformers for the GPU paths.

Mirror the reference's ``PbpQlp``, ``RandomizedSvd`` and ``CorUtv`` estimators
(estimators.py:81-157 on the shared ``_LowRankTransformer`` plumbing,
:31-78): ``fit`` factorizes on the GPU, ``components_`` holds the first
``n_components`` columns of the row-space basis transposed (P for PbP-QLP,
V for r_svd and cor_utv), ``singular_values_`` the estimates of
analysis.singular_value_estimates (|diag L|, resp. s), and ``transform`` /
``inverse_transform`` are the skinny products X·componentsᵀ and
Z·components run on libpbq's DMMA GEMM.  numpy in → numpy out; CUDA tensors
stay on the device.
"""
import numpy as np
import torch
from sklearn.base import BaseEstimator, TransformerMixin
from sklearn.exceptions import NotFittedError

from . import device as _dev
from . import exceptions as _exc
from .algorithms import pbp_qlp
from .linalg import HostMatrix
from .rsvd import r_svd
from .utv import cor_utv
from .validation import check_count

__all__ = ["PbpQlp", "RandomizedSvd", "CorUtv"]


def _gemm_nn(x, b):
    """x (m×k) · b (k×n) on the device with libpbq's GEMM."""
    ctx = _dev.context(x.device)
    return _dev.gemm(ctx, x, b, trans_a=False)


class _LowRankTransformer(BaseEstimator, TransformerMixin):
    """Shared plumbing (estimators.py:31-78); subclasses give
    ``_factorize(X, rank)``, ``_row_basis(f)`` and ``_spectrum(f)``."""

    def fit(self, X, y=None):
        h = HostMatrix(X, "X")
        if not h.all_finite():
            raise _exc.MatrixInputError("X contains non-finite entries")
        limit = min(h.shape)
        rank = check_count(self.n_components, "n_components", minimum=1, maximum=limit)
        self.n_components_ = rank
        self.factors_ = self._factorize(X, rank)
        basis = self._row_basis(self.factors_)
        spec = self._spectrum(self.factors_)
        if isinstance(basis, torch.Tensor):
            self.components_ = basis[:, :rank].T.contiguous()
            self.singular_values_ = spec[:rank].abs()
        else:
            self.components_ = np.ascontiguousarray(basis[:, :rank].T)
            self.singular_values_ = np.abs(spec)[:rank].copy()
        self.n_features_in_ = h.shape[1]
        return self

    def _check_fitted(self):
        if not hasattr(self, "factors_"):
            raise NotFittedError(f"{type(self).__name__} is not fitted yet; call fit first")

    def _apply(self, X, b, expect_cols, what):
        self._check_fitted()
        h = HostMatrix(X, "X")
        if not h.all_finite():
            raise _exc.MatrixInputError("X contains non-finite entries")
        if h.shape[1] != expect_cols:
            raise _exc.DimensionError(f"X has {h.shape[1]} columns but {what}")
        x = h.to_device(None)
        bd = torch.as_tensor(b).to(device=x.device, dtype=torch.float64)
        out = _gemm_nn(x, bd)
        if h.kind == "numpy":
            return out.cpu().numpy()
        return out if h.home is None or torch.device(h.home) == out.device else out.to(h.home)

    def transform(self, X):
        """Coordinates of each row of X in the learned row-space basis: X·componentsᵀ."""
        self._check_fitted()
        return self._apply(X, self.components_.T, self.n_features_in_,
                           f"the estimator was fitted with {self.n_features_in_}")

    def inverse_transform(self, X):
        """Lift coordinates back to the original column space: Z·components."""
        self._check_fitted()
        return self._apply(X, self.components_, self.n_components_,
                           f"the fitted basis has {self.n_components_} components")


class PbpQlp(_LowRankTransformer):
    """Randomized QLP factorization driven by a row-space sketch
    (estimators.py:81-108): ``fit`` computes Q L Pᵀ of rank
    ``n_components`` with ``q`` power iterations; ``inverse_transform(
    transform(X))`` reproduces the factorization's low-rank approximation."""

    def __init__(self, n_components, q=0, seed=0, reorthonormalize=True):
        self.n_components = n_components
        self.q = q
        self.seed = seed
        self.reorthonormalize = reorthonormalize

    def _factorize(self, X, rank):
        return pbp_qlp(X, rank, q=self.q, seed=self.seed, reorthonormalize=self.reorthonormalize)

    def _row_basis(self, f):
        return f.p_basis

    def _spectrum(self, f):
        return torch.diagonal(f.l) if isinstance(f.l, torch.Tensor) else np.diagonal(f.l)


class RandomizedSvd(_LowRankTransformer):
    """Randomized truncated SVD via a column-space sketch (estimators.py:111-126)."""

    def __init__(self, n_components, q=0, seed=0, reorthonormalize=True):
        self.n_components = n_components
        self.q = q
        self.seed = seed
        self.reorthonormalize = reorthonormalize

    def _factorize(self, X, rank):
        return r_svd(X, rank, q=self.q, seed=self.seed, reorthonormalize=self.reorthonormalize)

    def _row_basis(self, f):
        return f.v

    def _spectrum(self, f):
        return f.s


class CorUtv(_LowRankTransformer):
    """Randomized rank-revealing UTV via compressed orthogonal bases
    (estimators.py:128-157)."""

    def __init__(self, n_components, q=0, seed=0, pass_efficient=False, reorthonormalize=True):
        self.n_components = n_components
        self.q = q
        self.seed = seed
        self.pass_efficient = pass_efficient
        self.reorthonormalize = reorthonormalize

    def _factorize(self, X, rank):
        return cor_utv(X, rank, q=self.q, seed=self.seed, pass_efficient=self.pass_efficient,
                       reorthonormalize=self.reorthonormalize)

    def _row_basis(self, f):
        return f.v

    def _spectrum(self, f):
        return f.t_values
