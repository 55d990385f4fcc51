"""Compressed randomized UTV on the B200 kernels (the second
sibling path).

``cor_utv(a, d, q=0, seed=0, pass_efficient=False, reorthonormalize=True)``
follows /root/reference/pkg/src/pbpqlp/algorithms.py:306-363 call for call:

    Ω = gaussian_matrix(n2, d, seed)                 (bit-exact device sketch)
    f1 = A·Ω
    reorth:  Ū = orth(f1); q × [Ū = orth(AᵀŪ); Ū = orth(A·Ū)];  f2 = AᵀŪ
    else:    q × [f1 = A·(Aᵀ·f1)]; Ū = orth(f1); f2 = Aᵀ·f1; gram = Ūᵀ·f1
    V̄ = orth(f2)
    core = ŪᵀAV̄  (one more pass)   or, pass_efficient, f2ᵀV̄ (·pinv(gram)ᵀ)
    (Q_c, T, perm) = column_pivoted_qr(core);  U = Ū·Q_c;  V = V̄[:, perm]

Every pass over A, every orth, the pivot selection of the core's CPQR
(LAPACK dgeqp3's rule, cpqr_f64.cuh), its QR and the column gather run on
libpbq's sm_100a kernels, and so does the SVD of the k×d sample Gram factor
on the pass-efficient, non-reorthonormalized branch (``_transposed_pinv_apply``,
algorithms.py:295-303): libpbq's one-sided Jacobi core (pbq_jacobi_svd), like
r_svd's core SVD.
"""
from dataclasses import dataclass
from typing import Any, Optional

import torch

from . import device as _dev
from . import exceptions as _exc
from .algorithms import SketchRecord
from .linalg import HostMatrix, cpqr_device, from_device, warn_rank
from .validation import check_seed, check_sketch_params

__all__ = ["UtvFactors", "cor_utv", "cor_utv_flops", "PINV_RTOL"]

#: Relative singular-value cutoff of the pass-efficient pseudoinverse (algorithms.py:56).
PINV_RTOL = 1e-12


def cor_utv_flops(n1, n2, d, q, pass_efficient=False, reorthonormalize=True):
    """Algorithmic FLOPs of one cor_utv call, counted like pbp_qlp_flops
    (SURVEY.md §8d): 2·n1·n2·d per pass over A, LAPACK thin-QR counts for
    every orth and for the core's CPQR, the core and basis products."""
    k = min(n1, d)

    def qr(m, n):
        return 4.0 * m * n * n - 4.0 * n ** 3 / 3.0

    passes = 2 * q + 2 + (0 if pass_efficient else 1)
    f = passes * 2.0 * n1 * n2 * d
    if reorthonormalize:
        f += (q + 1) * qr(n1, k) + (q + 1) * qr(n2, k)
    else:
        f += qr(n1, k) + qr(n2, d) + 2.0 * n1 * k * d  # + the sample Gram Ūᵀ·f1
    f += 2.0 * n2 * d * d if pass_efficient else 2.0 * n1 * k * d  # core product
    f += qr(d, k) if d >= k else qr(k, d)  # CPQR of the k×d core
    f += 2.0 * n1 * k * k  # U = Ū·Q_c
    return f


@dataclass(frozen=True)
class UtvFactors:
    """Compressed factorization ``A ~ u @ t @ v.T`` with triangular ``t``
    (algorithms.py:145-168)."""

    u: Any
    t: Any
    v: Any
    pass_efficient: bool
    sketch: Optional[SketchRecord] = None
    pinv_truncated: bool = False

    @property
    def t_values(self):
        """Absolute diagonal of ``t``."""
        t = self.t
        if isinstance(t, torch.Tensor):
            return t.diagonal().abs()
        import numpy as np

        return np.abs(np.diagonal(t))

    def approx(self):
        """Reconstruct ``u @ t @ v.T``."""
        return self.u @ self.t @ self.v.T


def cor_utv(a, d, q=0, seed=0, pass_efficient=False, reorthonormalize=True, *, device=None):
    """Compressed randomized UTV factorization of ``a`` (algorithms.py:306-363)."""
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
    n_orth = (2 * q + 2) if reorthonormalize else 2
    flags = torch.zeros(2 + n_orth, dtype=torch.int32, device=dev)  # [nonfinite, sketch status, orth flags...]
    passes = 0

    def apply(x):
        nonlocal passes
        passes += 1
        return _dev.gemm(ctx, A, x, trans_a=False, nonfinite=flags[0:1] if passes == 1 else None)

    def apply_t(x):
        nonlocal passes
        passes += 1
        return _dev.gemm(ctx, A, x, trans_a=True)

    site = 2

    def orth_(m, final=True):
        """orth(m) on the device (first min(rows, cols) columns), rank flag → flags[site].
        ``final=False``: the result is only multiplied by A and orthonormalised
        again — basis-only (``pbq_orth_basis``: Q·T with T upper triangular,
        which leaves the next orth's Q factor unchanged)."""
        nonlocal site
        c = min(m.shape)
        truncated = m.shape[1] != c
        m = _dev.as_kernel_operand(m[:, :c]) if truncated else _dev.as_kernel_operand(m)
        if final or truncated:
            r = _dev.empty_matrix(c, c, dev)
            _dev.householder_qr_(ctx, m, r, want_q=True, rank_flag=flags[site:site + 1])
        else:
            m = _dev.orth_basis_(ctx, m, rank_flag=flags[site:site + 1])
        site += 1
        return m

    omega = _dev.gaussian(ctx, n2, d, seed, dev, status=flags[1:2])
    f1 = apply(omega)
    gram = None
    if reorthonormalize:
        ubar = orth_(f1, final=(q == 0))
        for it in range(q):  # _power_iterations(transpose_first=False): Aᵀ first, then A
            ubar = orth_(apply_t(ubar), final=False)
            ubar = orth_(apply(ubar), final=(it == q - 1))
        f2 = apply_t(ubar)
    else:
        for _ in range(q):
            f1 = apply(apply_t(f1))
        ubar = orth_(f1.clone())
        f2 = apply_t(f1)
        if pass_efficient:
            gram = _dev.gemm(ctx, ubar, f1, trans_a=True)  # Ūᵀ·f1, k×d
    vbar = orth_(f2.clone() if pass_efficient else f2)

    pinv_truncated = torch.zeros((), dtype=torch.bool, device=dev)
    if pass_efficient:
        core = _dev.gemm(ctx, f2, vbar, trans_a=True)  # f2ᵀ·V̄
        if gram is not None:
            # svd(gram) by the native Jacobi core on its k rows (k ≤ d):
            # G·gram = diag(s)·Y ⇒ u_g = Gᵀ, vh_g = Y (pbq_jacobi_svd)
            s_g, vh_g, g_g, jst = _dev.jacobi_svd(ctx, gram, accumulate=True, want_y=True)
            u_g = _dev.transpose(ctx, g_g)
            keep = s_g > PINV_RTOL * s_g[0]
            # s[0] == 0 keeps nothing: zero core, flagged (algorithms.py:298-299)
            inv = torch.where(keep, 1.0 / torch.where(keep, s_g, torch.ones_like(s_g)), torch.zeros_like(s_g))
            tmp = _dev.gemm(ctx, _dev.as_kernel_operand(vh_g), core, trans_a=False)  # vᵀ·core
            core = _dev.gemm(ctx, _dev.as_kernel_operand(u_g * inv), tmp, trans_a=False)
            pinv_truncated = (~keep).any()
    else:
        core = _dev.gemm(ctx, ubar, apply(vbar), trans_a=True)  # Ūᵀ·(A·V̄)

    q_c, t, perm = cpqr_device(ctx, _dev.as_kernel_operand(core))
    u = _dev.gemm(ctx, ubar, q_c, trans_a=False)
    v = _dev.gather_columns(ctx, vbar, perm)
    t = torch.triu(t)

    fl = flags.cpu().tolist()  # the one host read
    if fl[0]:
        raise _exc.MatrixInputError("a contains non-finite entries")
    if fl[1]:
        raise _exc.DeviceError("sketch generator overflow (internal error)")
    if gram is not None and int(jst[1].item()):
        raise _exc.ConvergenceError("cor_utv: the Jacobi SVD core of the pseudoinverse did not converge in 60 sweeps")
    for flag in fl[2:site]:
        warn_rank(flag, stacklevel=3)
    outs = [from_device(x, kind, home) for x in (u, t, v)]
    sketch = SketchRecord(omega, kind, seed, d, q, passes, home)
    return UtvFactors(outs[0], outs[1], outs[2], bool(pass_efficient), sketch, bool(pinv_truncated.item()))
