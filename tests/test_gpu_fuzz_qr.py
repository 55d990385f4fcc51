"""Randomized sweep of the QR entry point (`householder_qr` / `orth`,
linalg.py:96-165) under every method: random m ≥ n (1…300 columns, up to
3000 rows), condition numbers from 1 to 1e15 with graded, clustered and
rank-deficient spectra, against LAPACK (numpy.linalg.qr with the
reference's sign fix).  Every route is reached: the single-launch kernels
(n ≤ 128; 128 < n ≤ 256 with m ≤ 1024), the chain, the shifted route
(n ≥ 384 is not drawn here: it is covered by test_gpu_kernels.py), and the
Householder fallback, forced or on guard failure.

Checks: |QᵀQ − I| at LAPACK's level (≤ 64·u·√n), the reconstruction QR = A
to u·‖A‖, diag R ≥ 0 with exact zeros below, the rank flag equal to the
reference's rank test on LAPACK's R, and — for numerically full-rank
inputs — Q's columns within max(1e-10, 64·u·κ_j, 8× LAPACK's own noise on a
row-permuted input) of LAPACK's (κ_j = |R₀₀/R_jj|).  PBQ_FUZZ_CASES sets the count (default 60)."""
import os

import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import column_relative_error, oracle_qr, rank_flag

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def _matrix(seed):
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.choice([rng.integers(1, 33), rng.integers(33, 129), rng.integers(129, 301)]))
    m = int(max(n, rng.choice([n, n + rng.integers(0, 64), rng.integers(n, 3001)])))
    kind = rng.choice(["graded", "clustered", "deficient", "gaussian"])
    logk = float(rng.uniform(0, 15))
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if kind == "graded":
        s = np.logspace(0, -logk, n)
    elif kind == "clustered":
        s = np.where(np.arange(n) < n // 2, 1.0, 10.0 ** -logk)
    elif kind == "deficient":
        s = np.where(np.arange(n) < max(1, n // 3), 1.0, 0.0)
    else:
        return rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-3, 3), str(kind)
    return (u * s) @ v.T, str(kind)


@pytest.mark.parametrize("method", ["auto", "chain", "householder"])
@pytest.mark.parametrize("seed", range(int(os.environ.get("PBQ_FUZZ_CASES", "60"))))
def test_random_qr_matches_lapack(cuda, seed, method):
    from paper_2103_07245_b200 import device as D

    x, kind = _matrix(seed)
    m, n = x.shape
    ctx = D.context(cuda)
    ctx.set_qr_method({"auto": ctx.QR_AUTO, "chain": ctx.QR_CHOLQR_CHAIN, "householder": ctx.QR_HOUSEHOLDER}[method])
    try:
        t = D.empty_matrix(m, n, cuda)
        t.copy_(torch.from_numpy(x))
        r = D.empty_matrix(n, n, cuda)
        flag = torch.full((1,), -1, dtype=torch.int32, device=cuda)
        D.householder_qr_(ctx, t, r, rank_flag=flag)
        q, rr, fl = t.cpu().numpy(), r.cpu().numpy(), int(flag.item())
    finally:
        ctx.set_qr_method(ctx.QR_AUTO)
    qref, rref = oracle_qr(x)
    what = (m, n, kind, method)
    orth = np.abs(q.T @ q - np.eye(n)).max()
    assert orth <= 64 * U * np.sqrt(n) + 1e-15, (what, "orthogonality", orth)
    rec = np.abs(q @ rr - x).max() / max(np.abs(x).max(), 1e-300)
    assert rec <= 64 * U * np.sqrt(n), (what, "reconstruction", rec)
    assert np.all(np.diag(rr) >= 0) and np.array_equal(np.tril(rr, -1), np.zeros((n, n))), (what, "R structure")
    assert fl == rank_flag(rref), (what, "rank flag", fl, rank_flag(rref))
    if fl == 0:
        d = np.abs(np.diag(rref))
        kap = d[0] / d
        # LAPACK's own rounding noise: the same factorization of a row-permuted
        # input (clustered spectra make Q's columns far more sensitive than
        # R₀₀/R_jj suggests)
        perm = np.random.default_rng(seed).permutation(m)
        qalt, _ = oracle_qr(x[perm])
        noise = np.maximum.accumulate(column_relative_error(qalt[np.argsort(perm)], qref))
        tol = np.maximum(np.maximum(1e-10, 64 * U * kap), 8 * noise)
        err = column_relative_error(q, qref)
        assert np.all(err <= tol), (what, err.max(), int(np.argmax(err / tol)))
