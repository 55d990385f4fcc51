"""The second stage of PbP-QLP on the device, pbq_second_stage (reference
algorithms.py:256-257: (W, R̃) = householder_qr(Rᵀ), L = tril(R̃ᵀ)).

It runs the transpose + tall-QR chain; checked against the oracle's
sign-fixed LAPACK QR (linalg.py:96-115) of the same Rᵀ: W per column within
max(1e-10, 64·u·κ_j) and |diag L| within max(1e-10, 16·u·κ_j), κ_j = L₀₀/L_jj
(SURVEY §8 a9), plus exact structure (L lower triangular, diag L ≥ 0).
"""
import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import column_relative_error, oracle_qr

pytestmark = pytest.mark.gpu

U = 2.0**-53


def _r_factor(d, kind, rng):
    if kind == "graded":
        m = rng.standard_normal((3 * d, d)) * np.logspace(0, -4, d)
    elif kind == "lowrank":  # numerically rank-deficient tail (the config-3 shape: d beyond the signal rank)
        m = rng.standard_normal((3 * d, max(1, d // 2))) @ rng.standard_normal((max(1, d // 2), d))
        m += 1e-9 * rng.standard_normal((3 * d, d))
    else:
        m = rng.standard_normal((3 * d, d))
    return oracle_qr(m)[1]  # upper triangular, diag ≥ 0


@pytest.mark.parametrize("d", [1, 2, 17, 40, 100, 128, 160, 161, 256])
@pytest.mark.parametrize("kind", ["gauss", "graded", "lowrank"])
def test_second_stage_matches_oracle(cuda, d, kind):
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(1000 * d + len(kind))
    r = _r_factor(d, kind, rng)
    w_ref, rt_ref = oracle_qr(r.T)
    l_ref = np.tril(rt_ref.T)
    ctx = D.context(cuda)
    rd = D.empty_matrix(d, d, cuda)
    rd.copy_(torch.from_numpy(r))
    w, l = D.second_stage(ctx, rd)
    w, l = w.cpu().numpy(), l.cpu().numpy()
    assert np.array_equal(l, np.tril(l)) and np.all(np.diag(l) >= 0)
    ld = np.abs(np.diag(l_ref))
    kappa = ld[0] / np.maximum(ld, 1e-300)
    tol_l = np.maximum(1e-10, 16 * U * kappa)
    tol_w = np.maximum(1e-10, 64 * U * kappa)
    det = kappa < 1e8  # columns the factorization determines (the rest is a rank-deficient tail)
    assert np.all((np.abs(np.diag(l) - ld) <= tol_l * ld)[det])
    assert np.all((column_relative_error(w, w_ref) <= tol_w)[det])
    # W orthogonal and R = L·Wᵀ on every column
    assert np.abs(w.T @ w - np.eye(d)).max() < 1e-13
    assert np.linalg.norm(l @ w.T - r) <= 1e-13 * max(1.0, np.linalg.norm(r))


def test_second_stage_zero_and_identity(cuda):
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    for d in (5, 64):
        rd = D.empty_matrix(d, d, cuda)
        rd.copy_(torch.eye(d, dtype=torch.float64))
        w, l = D.second_stage(ctx, rd)
        assert np.abs(w.cpu().numpy() - np.eye(d)).max() < 1e-15 and np.abs(l.cpu().numpy() - np.eye(d)).max() < 1e-15
        rd.zero_()
        w, l = D.second_stage(ctx, rd)
        assert np.array_equal(l.cpu().numpy(), np.zeros((d, d)))  # zero R: R̃ = 0
        wz = w.cpu().numpy()
        assert np.abs(wz.T @ wz - np.eye(d)).max() < 1e-13  # any orthogonal W (the reference's is I)
