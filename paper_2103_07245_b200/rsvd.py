"""Randomized SVD on the B200 kernels (the first sibling path).

``r_svd(a, d, q=0, seed=0, reorthonormalize=True)`` follows
/root/reference/pkg/src/pbpqlp/algorithms.py:263-292 call for call:

    Ω = gaussian_matrix(n2, d, seed)              (linalg.py:83-93; bit-exact device sketch)
    f = A·Ω                                        (pass 1, fused Inf/NaN scan of A)
    reorth:  Ū = orth(f); q × [Ū = orth(AᵀŪ); Ū = orth(A·Ū)]     (_power_iterations,
    else:    q × [f = A·(Aᵀ·f)]; Ū = orth(f)                      transpose_first=False)
    g = (AᵀŪ)ᵀ                                      (one pass)
    U_c, s, V = svd_full(g);  u = Ū·U_c            (linalg.py:131-139)

The A passes and every ``orth`` run on libpbq's sm_100a kernels (DMMA GEMM,
Cholesky-QR2 with Householder fallback).  The SVD of the k×n2 matrix g is
reduced to a k×k core: h = AᵀŪ = Q_h·R_h (libpbq QR), so g = R_hᵀ·Q_hᵀ and
svd(R_hᵀ) = U_c·diag(s)·W_cᵀ gives v = Q_h·W_c.  The k×k SVD (k ≤ d) is
libpbq's one-sided Jacobi core (pbq_jacobi_svd, svd_f64.cuh: one thread-block
cluster, the vectors in registers), preconditioned by one more k×k QR
(R_hᵀ = W·R̃, pbq_second_stage).  As in the reference, singular vectors
carry arbitrary signs; u_j and v_j are defined up to a joint sign.  When
d > n1 the reference's ``orth`` of the n1×d sample returns n1 columns (the Householder Q is fixed by the first
min(n1, d) columns), and so does this path.
"""
from dataclasses import dataclass
from typing import Any, Optional

import torch

from . import device as _dev
from . import exceptions as _exc
from .algorithms import SketchRecord
from .linalg import HostMatrix, from_device, warn_rank
from .validation import check_seed, check_sketch_params

__all__ = ["RsvdFactors", "r_svd", "r_svd_flops"]


def r_svd_flops(n1, n2, d, q, reorthonormalize=True):
    """Algorithmic FLOPs of one r_svd call, counted like pbp_qlp_flops
    (SURVEY.md §8d): 2q+2 passes over A, LAPACK thin-QR counts for every
    orth, the k×k core (QR of the n2×k h, 21k³ for the dense SVD with
    vectors, and the two basis products)."""
    k = min(n1, d)

    def qr(m, n):
        return 4.0 * m * n * n - 4.0 * n ** 3 / 3.0

    f = (2 * q + 2) * 2.0 * n1 * n2 * d
    f += ((q + 1) * qr(n1, k) + q * qr(n2, k)) if reorthonormalize else qr(n1, k)
    f += qr(n2, k) + 21.0 * k ** 3 + 2.0 * n1 * k * k + 2.0 * n2 * k * k
    return f


@dataclass(frozen=True)
class RsvdFactors:
    """Rank-``d`` SVD estimate ``u @ diag(s) @ v.T`` (algorithms.py:131-142)."""

    u: Any
    s: Any
    v: Any
    sketch: Optional[SketchRecord] = None

    def approx(self):
        return (self.u * self.s) @ self.v.T


def r_svd(a, d, q=0, seed=0, reorthonormalize=True, *, device=None):
    """Randomized SVD of ``a`` with rank parameter ``d`` (algorithms.py:263-292)."""
    ha = HostMatrix(a, "a")
    n1, n2 = ha.shape
    try:
        d, q = check_sketch_params(d, q, n2)
    except _exc.ParameterError:
        if not ha.all_finite():
            raise _exc.MatrixInputError("a contains non-finite entries") from None
        raise
    seed = check_seed(seed)
    kind, home = ha.kind, ha.home
    A = ha.to_device(device)
    dev = A.device
    ctx = _dev.context(dev)
    k = min(n1, d)
    n_orth = (2 * q + 1) if reorthonormalize else 1
    flags = torch.zeros(2 + n_orth, dtype=torch.int32, device=dev)  # [nonfinite, sketch status, orth flags...]

    omega = _dev.gaussian(ctx, n2, d, seed, dev, status=flags[1:2])
    f = _dev.empty_matrix(n1, d, dev)
    _dev.gemm(ctx, A, omega, trans_a=False, out=f, nonfinite=flags[0:1])  # pass 1: f = A·Ω

    site = 2

    def orth_(m, final=True):
        """orth(m) on the device (first k columns), rank flag → flags[site].
        ``final=False``: the result is only multiplied by A and orthonormalised
        again — basis-only (``pbq_orth_basis``: Q·T with T upper triangular,
        which leaves the next orth's Q factor unchanged)."""
        nonlocal site
        m = _dev.as_kernel_operand(m[:, :k]) if m.shape[1] != k else m
        if final or m.shape[1] != k:
            r = _dev.empty_matrix(k, k, dev)
            _dev.householder_qr_(ctx, m, r, want_q=True, rank_flag=flags[site:site + 1])
        else:
            m = _dev.orth_basis_(ctx, m, rank_flag=flags[site:site + 1])
        site += 1
        return m

    t = _dev.empty_matrix(n2, k, dev)
    if reorthonormalize:
        ubar = orth_(f, final=(q == 0))
        for it in range(q):  # transpose_first=False: A.T first, then A
            _dev.gemm(ctx, A, ubar, trans_a=True, out=t)
            tb = orth_(t, final=False)
            ubar_next = _dev.empty_matrix(n1, k, dev)
            _dev.gemm(ctx, A, tb, trans_a=False, out=ubar_next)
            ubar = orth_(ubar_next, final=(it == q - 1))
    else:
        tt = _dev.empty_matrix(n2, d, dev)
        for _ in range(q):
            _dev.gemm(ctx, A, f, trans_a=True, out=tt)
            _dev.gemm(ctx, A, tt, trans_a=False, out=f)
        ubar = orth_(f)

    # g = (AᵀŪ)ᵀ, one pass; its SVD through the QR of h = AᵀŪ (k ≤ d ≤ n2)
    h = _dev.empty_matrix(n2, k, dev)
    _dev.gemm(ctx, A, ubar, trans_a=True, out=h)
    rh = _dev.empty_matrix(k, k, dev)
    _dev.householder_qr_(ctx, h, rh, want_q=True)  # h ← Q_h (the reference does not warn here)
    # svd(R_hᵀ): first the QLP step (W, R̃) = qr(R_hᵀ) (pbq_second_stage; the
    # diagonal of R̃ tracks the singular values, so its rows are graded like
    # them — the QR preconditioning of one-sided Jacobi, Drmač & Veselić
    # 2008), then the native one-sided Jacobi core on the rows of R̃:
    # G·R̃ = diag(s)·Y ⇒ R_hᵀ = W·R̃ = (W·Gᵀ)·diag(s)·Y, so U_c = W·Gᵀ and
    # W_c = Yᵀ (pbq_jacobi_svd, svd_f64.cuh)
    w, l = _dev.second_stage(ctx, rh)  # l = tril(R̃ᵀ)
    s, y, g, jst = _dev.jacobi_svd(ctx, _dev.transpose(ctx, l), accumulate=True, want_y=True, precondition=False)
    uc = _dev.gemm(ctx, w, _dev.transpose(ctx, g), trans_a=False)
    u = _dev.gemm(ctx, ubar, uc, trans_a=False)
    v = _dev.gemm(ctx, h, _dev.transpose(ctx, y), trans_a=False)

    fl = flags.cpu().tolist()  # the one host read
    if fl[0]:
        raise _exc.MatrixInputError("a contains non-finite entries")
    if fl[1]:
        raise _exc.DeviceError("sketch generator overflow (internal error)")
    if int(jst[1].item()):
        raise _exc.ConvergenceError("r_svd: the Jacobi SVD core did not converge in 60 sweeps")
    for flag in fl[2:]:
        warn_rank(flag, stacklevel=3)
    outs = [from_device(x, kind, home) for x in (u, s.contiguous(), v)]
    sketch = SketchRecord(omega, kind, seed, d, q, 2 * q + 2, home)
    return RsvdFactors(outs[0], outs[1], outs[2], sketch)
