"""Callers of the PbP-QLP path on the GPU.

Mirrors the reference's dispatcher and error helpers for the algorithm this
package implements:

* ``factorize(a, "pbp_qlp" | "r_svd" | "cor_utv" | "cpqr", d, ...)`` ↔ analysis.py:135-157
* ``low_rank_approx(factors, rank)``         ↔ analysis.py:159-193
* ``spectral_norm(m)``                        ↔ linalg.py:194-207 (+ _power_norm :168-191)
* ``residual_spectral_norm(a, f, rank)``      ‖A − approx‖₂ without forming the residual
* ``error_curve(a, alg, d_values, ...)``       ↔ analysis.py:213-247

The factorization and the Frobenius residual run on libpbq's sm_100a
kernels (the fused one-pass residual).  The spectral norm of a
residual follows the reference's algorithm exactly: a dense singular value
up to 2000 in the larger dimension, else power iteration on the Gram
operator from the seeded start vector gaussian_matrix(n, 1, seed=0x5EED),
relative tolerance 1e-10, at most 5000 iterations.  Its matrix-vector
products use torch on the device; it is an analysis helper, not the hot path.
The exact ``svd`` and the deterministic ``pqlp`` are outside this package's
scope and raise.
"""
import math

import numpy as np
import torch

from . import exceptions as _exc
from .algorithms import QlpFactors, pbp_qlp, residual_norms
from .rsvd import RsvdFactors, r_svd
from .linalg import HostMatrix, QrFactors, column_pivoted_qr, gaussian_matrix
from .utv import UtvFactors, cor_utv
from .validation import check_index_range

__all__ = ["ALGORITHMS", "GPU_ALGORITHMS", "factorize", "low_rank_approx", "spectral_norm",
           "residual_spectral_norm", "error_curve"]

ALGORITHMS = ("svd", "cpqr", "pqlp", "r_svd", "cor_utv", "pbp_qlp")  # analysis.py:53-55
GPU_ALGORITHMS = ("cpqr", "r_svd", "cor_utv", "pbp_qlp")
DETERMINISTIC_ALGORITHMS = ("svd", "cpqr", "pqlp")  # analysis.py:56
DENSE_NORM_LIMIT = 2000  # linalg.py:40
POWER_RTOL = 1e-10       # linalg.py:43
POWER_MAXITER = 5000     # linalg.py:44
POWER_SEED = 0x5EED      # linalg.py:172


def _check_algorithm(algorithm):
    if algorithm not in ALGORITHMS:
        raise _exc.ParameterError(f"unknown algorithm id {algorithm!r}; expected one of {ALGORITHMS}")
    if algorithm not in GPU_ALGORITHMS:
        raise _exc.ParameterError(
            f"algorithm {algorithm!r} is outside the B200 path of this package (implemented: {GPU_ALGORITHMS})"
        )


def _check_finite(h, name):
    if not h.all_finite():
        raise _exc.MatrixInputError(f"{name} contains non-finite entries")


def factorize(a, algorithm, d, q=0, seed=0, reorthonormalize=True):
    """Run one algorithm selected by id (analysis.py:135-157); ``a`` is
    validated first, as in the reference."""
    if algorithm not in GPU_ALGORITHMS:
        _check_finite(HostMatrix(a, "a"), "a")
        _check_algorithm(algorithm)
    if algorithm == "cpqr":
        _check_finite(HostMatrix(a, "a"), "a")
        return column_pivoted_qr(a)
    if algorithm == "r_svd":
        return r_svd(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize)
    if algorithm == "cor_utv":
        return cor_utv(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize)
    return pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize)


def low_rank_approx(factors, rank=None):
    """Reconstruction, optionally truncated (analysis.py:170-193) for the
    factor types of this package."""
    if isinstance(factors, QlpFactors):
        return factors.approx(rank)
    if isinstance(factors, RsvdFactors):
        if rank is None:
            return factors.approx()
        rank = check_index_range(rank, "rank", 1, factors.s.shape[0])
        return (factors.u[:, :rank] * factors.s[:rank]) @ factors.v[:, :rank].T
    if isinstance(factors, UtvFactors):
        if rank is None:
            return factors.approx()
        rank = check_index_range(rank, "rank", 1, factors.t.shape[0])
        return factors.u[:, :rank] @ factors.t[:rank, :rank] @ factors.v[:, :rank].T
    if isinstance(factors, QrFactors):  # analysis.py:159-167 (_pivoted_qr_approx)
        q, r, perm = factors
        rank = r.shape[0] if rank is None else check_index_range(rank, "rank", 1, r.shape[0])
        cols = q[:, :rank] @ r[:rank, :]
        if perm is None:
            return cols
        out = cols.clone() if isinstance(cols, torch.Tensor) else np.empty((q.shape[0], r.shape[1]))
        out[:, perm] = cols
        return out
    raise _exc.ParameterError(f"cannot reconstruct from factors of type {type(factors).__name__}")


def _device_of(*xs):
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    return torch.device("cuda", torch.cuda.current_device())


def _power_norm(apply, apply_t, n, rtol=POWER_RTOL, maxiter=POWER_MAXITER, device=None):
    """linalg.py:168-191 with the operator given by two device callables."""
    v = gaussian_matrix(n, 1, seed=POWER_SEED, device=device, as_tensor=True).reshape(-1).clone()
    v /= torch.linalg.vector_norm(v)
    estimate = 0.0
    for _ in range(maxiter):
        w = apply(v)
        nw = float(torch.linalg.vector_norm(w))
        if nw == 0.0:
            return 0.0
        v = apply_t(w)
        nv = float(torch.linalg.vector_norm(v))
        if nv == 0.0:
            return 0.0
        v /= nv
        new_estimate = nv / nw
        if abs(new_estimate - estimate) <= rtol * max(new_estimate, 1e-300):
            return new_estimate
        estimate = new_estimate
    raise _exc.ConvergenceError(
        f"power iteration did not reach relative tolerance {rtol:g} within {maxiter} iterations", estimate=estimate
    )


def spectral_norm(m, *, device=None):
    """Largest singular value of ``m`` (linalg.py:194-207)."""
    h = HostMatrix(m, "m")
    _check_finite(h, "m")
    t = h.to_device(device)
    if max(t.shape) <= DENSE_NORM_LIMIT:
        return float(torch.linalg.svdvals(t)[0])
    return float(_power_norm(lambda x: t @ x, lambda x: t.T @ x, t.shape[1], device=t.device))


def residual_spectral_norm(a, factors, rank=None, *, device=None):
    """‖A − approx(rank)‖₂: the reference's spectral_norm(a − approx) without
    forming the residual on the power-iteration path."""
    t = HostMatrix(a, "a").to_device(device)
    dev = t.device

    def on_dev(x):
        return torch.as_tensor(x).to(device=dev, dtype=torch.float64)

    if isinstance(factors, RsvdFactors):
        kmax = factors.s.shape[0]
        k = kmax if rank is None else check_index_range(rank, "rank", 1, kmax)
        q, l, p = on_dev(factors.u)[:, :k], torch.diag(on_dev(factors.s)[:k]), on_dev(factors.v)[:, :k]
    elif isinstance(factors, UtvFactors):
        kmax = factors.t.shape[0]
        if rank is None:
            q, l, p = on_dev(factors.u), on_dev(factors.t), on_dev(factors.v)
        else:
            k = check_index_range(rank, "rank", 1, kmax)
            q, l, p = on_dev(factors.u)[:, :k], on_dev(factors.t)[:k, :k], on_dev(factors.v)[:, :k]
    else:
        kmax = factors.l.shape[0]
        k = kmax if rank is None else check_index_range(rank, "rank", 1, kmax)
        q, l, p = on_dev(factors.q_basis)[:, :k], on_dev(factors.l)[:k, :k], on_dev(factors.p_basis)[:, :k]
    if max(t.shape) <= DENSE_NORM_LIMIT:
        return float(torch.linalg.svdvals(t - q @ l @ p.T)[0])
    return float(_power_norm(lambda x: t @ x - q @ (l @ (p.T @ x)),
                             lambda x: t.T @ x - p @ (l.T @ (q.T @ x)), t.shape[1], device=dev))


def error_curve(a, alg, d_values, q=0, seed=0, reorthonormalize=True):
    """Reconstruction error for each sampling size in ``d_values``
    (analysis.py:213-247): one record {d, spectral_error, frobenius_error}
    per point, each from a fresh factorization with the same ``seed``."""
    h = HostMatrix(a, "a")
    _check_finite(h, "a")
    t = h.to_device(None)
    limit = min(t.shape)
    d_list = [check_index_range(d, "d", 1, limit) for d in d_values]
    if not d_list:
        raise _exc.ParameterError("d_values must contain at least one sampling size")
    _check_algorithm(alg)
    records = []
    if alg in DETERMINISTIC_ALGORITHMS:  # factored once, truncated per point (analysis.py:229-236)
        from . import device as _dev

        base = column_pivoted_qr(t)
        ctx = _dev.context(t.device)
        a_perm = _dev.gather_columns(ctx, t, base.perm)  # ‖A − approx‖ = ‖A[:, perm] − Q_d R_d‖
        for d in d_list:
            trunc = RsvdFactors(base.q[:, :d], torch.ones(d, dtype=torch.float64, device=t.device),
                                base.r[:d, :].T, None)
            fro, _ = residual_norms(a_perm, trunc)
            records.append({"d": d, "spectral_error": residual_spectral_norm(a_perm, trunc), "frobenius_error": fro})
        return records
    for d in d_list:
        fac = factorize(t, alg, d, q=q, seed=seed, reorthonormalize=reorthonormalize)
        fro, _ = residual_norms(t, fac)
        records.append({"d": d, "spectral_error": residual_spectral_norm(t, fac), "frobenius_error": fro})
    return records
