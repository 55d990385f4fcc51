"""The native Jacobi SVD core (svd_f64.cuh, pbq_jacobi_svd) against LAPACK
(numpy.linalg.svd — the reference's `svd_full`, linalg.py:131-139): sorted
singular values within max(1e-13·σ₀-relative, …) of LAPACK's, orthonormal
factors, reconstruction X = Gᵀ·diag(s)·Y to rounding, sign-aligned singular
vectors within the gap-aware bound u·σ₀/gap_j, for both kernels (register /
cluster and L2-resident), graded and clustered spectra, zero rows and odd n."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def _graded(n, L, decades, seed):
    rng = np.random.default_rng(seed)
    qa, _ = np.linalg.qr(rng.standard_normal((n, n)))
    qb, _ = np.linalg.qr(rng.standard_normal((L, n)))
    return (qa * np.logspace(0, -decades, n)) @ qb.T


def _check(x, s, y, g, status, max_sweeps=20):
    n, L = x.shape
    s, y, g = s.cpu().numpy(), y.cpu().numpy(), g.cpu().numpy()
    sweeps, noconv = status.cpu().tolist()
    assert noconv == 0 and 1 <= sweeps <= max_sweeps
    ref = np.linalg.svd(x, compute_uv=False)
    assert np.all(np.diff(s) <= 0)
    s0 = max(ref[0], 1e-300)
    assert np.all(np.abs(s - ref) <= 64 * n * U * s0), np.max(np.abs(s - ref)) / s0
    assert np.abs(y @ y.T - np.eye(n)).max() < 64 * n * U
    assert np.abs(g @ g.T - np.eye(n)).max() < 64 * n * U
    rec = g.T @ (s[:, None] * y)
    assert np.abs(rec - x).max() <= 64 * n * U * max(s0, np.abs(x).max())
    return sweeps


@pytest.mark.parametrize("n,L", [(1, 1), (2, 5), (7, 7), (40, 40), (33, 90), (128, 128), (256, 256), (255, 300),
                                 (256, 512), (100, 700)])
@pytest.mark.parametrize("kernel", ["reg", "l2"])
def test_jacobi_svd_matches_lapack(cuda, monkeypatch, n, L, kernel):
    from paper_2103_07245_b200 import device as D

    if kernel == "l2":
        monkeypatch.setenv("PBQ_JACOBI_L2", "1")
    x = _graded(n, L, 8, n * 31 + L)
    s, y, g, st = D.jacobi_svd(D.context(cuda), torch.from_numpy(x).to(cuda))
    _check(x, s, y, g, st)


@pytest.mark.parametrize("n", [300, 600])
def test_jacobi_svd_large_l2_path(cuda, n):
    """n > 256 pairs beyond the register kernel: the L2-resident kernel."""
    from paper_2103_07245_b200 import device as D

    x = _graded(n, n, 10, n)
    s, y, g, st = D.jacobi_svd(D.context(cuda), torch.from_numpy(x).to(cuda))
    _check(x, s, y, g, st)


@pytest.mark.parametrize("n,L", [(40, 40), (128, 160), (255, 300)])
def test_jacobi_svd_unpreconditioned(cuda, n, L):
    """The plain core (no QR preconditioning) on graded rows: cyclic
    one-sided Jacobi needs 25–45 sweeps there, within its 60-sweep limit."""
    from paper_2103_07245_b200 import device as D

    x = _graded(n, L, 8, n * 31 + L)
    s, y, g, st = D.jacobi_svd(D.context(cuda), torch.from_numpy(x).to(cuda), precondition=False)
    _check(x, s, y, g, st, max_sweeps=60)


def test_jacobi_svd_vectors_and_special_inputs(cuda):
    """Singular vectors match LAPACK's up to sign within u·σ₀/gap_j; exactly
    zero rows and rank deficiency give an orthonormal completion; the result is
    bitwise reproducible."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    x = _graded(64, 80, 6, 5)
    s, y, g, st = D.jacobi_svd(ctx, torch.from_numpy(x).to(cuda))
    u_ref, s_ref, vt_ref = np.linalg.svd(x, full_matrices=False)
    yv, gv = y.cpu().numpy(), g.cpu().numpy()
    gap = np.minimum(np.abs(np.diff(s_ref, prepend=np.inf)), np.abs(np.diff(s_ref, append=-np.inf)))
    for j in range(64):
        sgn = np.sign(yv[j] @ vt_ref[j])
        bound = 256 * U * s_ref[0] / gap[j] + 1e-14
        assert np.linalg.norm(sgn * yv[j] - vt_ref[j]) <= bound
        assert np.linalg.norm(sgn * gv[j] - u_ref[:, j]) <= bound
    s2, y2, g2, _ = D.jacobi_svd(ctx, torch.from_numpy(x).to(cuda))
    assert torch.equal(s, s2) and torch.equal(y, y2) and torch.equal(g, g2)
    # zero rows and an exactly rank-2 matrix
    z = np.zeros((6, 9))
    z[1] = np.arange(9.0)
    z[4] = np.arange(9.0)[::-1]
    s, y, g, st = D.jacobi_svd(ctx, torch.from_numpy(z).to(cuda))
    _check(z, s, y, g, st)
    assert np.count_nonzero(s.cpu().numpy()) == 2
    s, y, g, st = D.jacobi_svd(ctx, torch.zeros((5, 5), dtype=torch.float64, device=cuda))
    _check(np.zeros((5, 5)), s, y, g, st)
