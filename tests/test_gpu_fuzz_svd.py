"""Randomized sweep of the Jacobi SVD core (pbq_jacobi_svd, svd_f64.cuh)
and of the sibling paths built on it.

* Core: random n×L (1 ≤ n ≤ 300, n ≤ L ≤ 700) with graded, clustered,
  repeated and rank-deficient spectra, both kernels (register/cluster and
  grid), with and without QR preconditioning: sorted singular values within
  64·n·u·σ₀ of LAPACK's, orthonormal Y and G, and X = Gᵀ·diag(s)·Y to
  rounding — the contract of svd_full (linalg.py:131-139) up to LAPACK's own
  accuracy class.
* r_svd (algorithms.py:263-292): random shapes and d, q, reorthonormalize
  against oracle_r_svd: singular values (σ_j ≥ 1e-6·σ₀) within
  max(1e-10, 16·u·σ₀/σ_j, 8× the reference's own noise on a row-permuted A)
  relative, and the rank-d approximation u·diag(s)·vᵀ within max(1e-10,
  8× that noise) of the reference's, in Frobenius norm relative to ‖A‖.
  Non-reorthonormalized cases with q ≥ 1 whose trailing sample directions
  sit below rounding must instead be at least as good an approximation as
  the reference's (see test_random_r_svd).
PBQ_FUZZ_CASES sets the count (default 30)."""
import os

import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import oracle_r_svd

pytestmark = pytest.mark.gpu
U = 2.0 ** -53
N = int(os.environ.get("PBQ_FUZZ_CASES", "30"))


def _spectrum(rng, n):
    kind = rng.choice(["graded", "clustered", "repeated", "deficient", "flat"])
    logk = float(rng.uniform(0, 12))
    if kind == "graded":
        s = np.logspace(0, -logk, n)
    elif kind == "clustered":
        s = np.where(np.arange(n) < n // 2, 1.0, 10.0 ** -logk) * (1 + 1e-3 * rng.standard_normal(n))
    elif kind == "repeated":
        s = np.repeat(np.logspace(0, -logk, max(1, n // 4) + 1), 4)[:n]
    elif kind == "deficient":
        s = np.where(np.arange(n) < max(1, n // 3), 1.0, 0.0)
    else:
        s = np.ones(n)
    return np.abs(s), str(kind)


@pytest.mark.parametrize("seed", range(N))
@pytest.mark.parametrize("kernel,pre", [("reg", True), ("reg", False), ("grid", True)])
def test_random_jacobi_svd(cuda, monkeypatch, seed, kernel, pre):
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(1, 301))
    L = int(rng.integers(n, max(n + 1, 701)))
    s_true, kind = _spectrum(rng, n)
    qa, _ = np.linalg.qr(rng.standard_normal((n, n)))
    qb, _ = np.linalg.qr(rng.standard_normal((L, n)))
    x = (qa * s_true) @ qb.T * 10.0 ** rng.uniform(-5, 5)
    if kernel == "grid":
        monkeypatch.setenv("PBQ_JACOBI_L2", "1")
    s, y, g, st = D.jacobi_svd(D.context(cuda), D.as_kernel_operand(torch.from_numpy(x).to(cuda)), precondition=pre)
    s, y, g = s.cpu().numpy(), y.cpu().numpy(), g.cpu().numpy()
    sweeps, noconv = st.cpu().tolist()
    what = (n, L, kind, kernel, pre, sweeps)
    assert noconv == 0, what
    ref = np.linalg.svd(x, compute_uv=False)
    s0 = max(ref[0], 1e-300)
    assert np.all(np.diff(s) <= 0), what
    assert np.abs(s - ref).max() <= 64 * n * U * s0, (what, np.abs(s - ref).max() / s0)
    assert np.abs(y @ y.T - np.eye(n)).max() <= 64 * np.sqrt(n) * U * 8, (what, "Y")
    assert np.abs(g @ g.T - np.eye(n)).max() <= 64 * np.sqrt(n) * U * 8, (what, "G")
    assert np.abs(g.T @ (s[:, None] * y) - x).max() <= 64 * n * U * max(s0, np.abs(x).max()), (what, "recon")


@pytest.mark.parametrize("seed", range(N))
def test_random_r_svd(cuda, seed):
    from paper_2103_07245_b200.rsvd import r_svd

    rng = np.random.default_rng(8000 + seed)
    n1, n2 = int(rng.integers(30, 1500)), int(rng.integers(30, 1500))
    kmin = min(n1, n2)
    d = int(rng.integers(1, min(kmin, 260) + 1))
    q = int(rng.integers(0, 3))
    reorth = bool(rng.random() < 0.8)
    r = int(min(kmin, d + rng.integers(0, 30)))
    u, _ = np.linalg.qr(rng.standard_normal((n1, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n2, r)))
    a = (u * np.exp(-np.arange(r) / float(rng.choice([5.0, 30.0, 1e9])))) @ v.T + 1e-8 * rng.standard_normal((n1, n2))
    sd = int(rng.integers(0, 2**31))
    got = r_svd(a, d, q=q, seed=sd, reorthonormalize=reorth)
    ref = oracle_r_svd(a, d, q=q, seed=sd, reorthonormalize=reorth)
    # the reference's own rounding noise: the same math on a row-permuted A
    # (r_svd's sketch Ω is n2×d, so permuting A's rows leaves the sketch alone)
    perm = np.random.default_rng(seed).permutation(n1)
    alt = oracle_r_svd(a[perm], d, q=q, seed=sd, reorthonormalize=reorth)
    s, sr, sa = np.asarray(got.s), np.asarray(ref["s"]), np.asarray(alt["s"])
    what = (a.shape, d, q, reorth)
    rel = lambda x: np.abs(x - sr) / np.maximum(sr, 1e-300)  # noqa: E731
    tol = np.maximum(np.maximum(1e-10, 16 * U * sr[0] / np.maximum(sr, 1e-300)), 8 * np.maximum.accumulate(rel(sa)))
    det = sr >= 1e-6 * sr[0]
    na = np.linalg.norm(a)
    app = (np.asarray(got.u) * s) @ np.asarray(got.v).T
    app_ref = (ref["u"] * sr) @ ref["v"].T
    app_alt = (alt["u"] * sa) @ alt["v"].T
    noise = np.linalg.norm(app_alt[np.argsort(perm)] - app_ref) / na
    err = np.linalg.norm(app - app_ref) / na
    if np.all(rel(s)[det] <= tol[det]) and err <= max(1e-10, 8 * noise):
        return
    # Where the sample (AAᵀ)^q·A·Ω keeps a direction only below rounding (the
    # non-reorthonormalized branch: σ_j^(2q+1)/σ₀^(2q+1) < u), the reference
    # and its row-permuted twin lose it the same way and agree with each
    # other, while the device's different (blocked) summation keeps a
    # different part of it.  Then the device must be an approximation at
    # least as good as the reference's: σ_j no farther from A's true σ_j
    # (to 2%), never above it (interlacing), and ‖A − u·diag(s)·vᵀ‖ no
    # larger (to 2%).
    assert not reorth and q >= 1, (what, (rel(s) / tol)[det].max(), err, noise)
    st = np.linalg.svd(a, compute_uv=False)[:d]
    dist = lambda x: np.abs(x - st) / np.maximum(st, 1e-300)  # noqa: E731
    assert np.all(dist(s)[det] <= 1.02 * dist(sr)[det] + tol[det]), (what, "farther from σ(A)")
    assert np.all(s <= st * (1 + 64 * U * d) + 64 * U * st[0]), (what, "above σ(A)")
    res = np.linalg.norm(a - app) / na
    res_ref = np.linalg.norm(a - app_ref) / na
    assert res <= 1.02 * res_ref + 1e-13, (what, res, res_ref)
