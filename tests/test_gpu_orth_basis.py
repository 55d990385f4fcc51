"""Basis-only orth (``pbq_orth_basis``) and its use inside the pipeline.

The reference's power iterations call ``orth`` on every intermediate product
(/root/reference/pkg/src/pbpqlp/algorithms.py:196-205).  An intermediate basis
is only multiplied by A and orthonormalised again, and the thin QR is
invariant under right-multiplication by an upper-triangular matrix T with
positive diagonal: qr(A·Q·T) has the Q factor of qr(A·Q).  ``pbq_orth_basis``
returns B = Q·T (one Cholesky-QR pass) — these tests pin exactly that
structure against LAPACK, and that the pipeline's factors do not move when the
switch is flipped.
"""
import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp, oracle_qr

pytestmark = pytest.mark.gpu


def _dev_matrix(x, dev):
    from paper_2103_07245_b200 import device as D

    t = D.empty_matrix(x.shape[0], x.shape[1], dev)
    t.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return t


def _basis(ctx, cuda, x):
    from paper_2103_07245_b200 import device as D

    flag = torch.full((1,), -1, dtype=torch.int32, device=cuda)
    out = D.orth_basis_(ctx, _dev_matrix(x, cuda), rank_flag=flag)
    torch.cuda.synchronize()
    return out.cpu().numpy(), int(flag.item())


def _graded(rng, m, n, kappa):
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (u * np.logspace(0, -np.log10(kappa), n)) @ v.T


# chain route: n ≤ 128 with m beyond the single-launch kernel, n > 128 with m > 1024;
# (2000, 512): the extended chain; the small shapes take the in-place routes
@pytest.mark.parametrize("m,n", [(12000, 96), (4000, 200), (20000, 256), (10000, 255), (2000, 512), (1000, 40),
                                 (600, 256), (64, 64)])
def test_basis_is_q_times_upper_triangular(cuda, m, n):
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(m + n)
    x = rng.standard_normal((m, n)) * np.logspace(0, -3, n)
    b, flag = _basis(ctx, cuda, x)
    q, _ = oracle_qr(x)
    t = q.T @ b
    assert flag == 0
    assert np.abs(np.tril(t, -1)).max() < 1e-12, "T is not upper triangular"
    assert np.all(np.diag(t) > 0.99)
    assert np.abs(t.T @ t - np.eye(n)).max() < 1e-3, "B is not near-orthonormal"
    # range(B) = range(Q) and the QR of B returns Q itself
    assert np.abs(b - q @ t).max() < 1e-12
    qb, _ = oracle_qr(b)
    assert column_relative_error(qb, q).max() < 1e-11


def test_next_orth_is_unchanged(cuda):
    """orth(A·B) equals orth(A·Q): what the power iterations rely on."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3000, 5000))
    c = _graded(rng, 5000, 160, 1e4)
    b, _ = _basis(ctx, cuda, c)
    q, _ = oracle_qr(c)
    nxt = D.gemm(ctx, _dev_matrix(a, cuda), _dev_matrix(b, cuda), trans_a=False)
    D.householder_qr_(ctx, nxt)
    ref, _ = oracle_qr(a @ q)
    assert column_relative_error(nxt.cpu().numpy(), ref).max() < 1e-10


def test_guard_failure_hands_over_the_full_qr(cuda):
    """κ beyond the Cholesky guard: the in-place fallback runs and its Q is copied out."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(4)
    stats = torch.zeros(4, dtype=torch.int32, device=cuda)
    ctx.cholqr_stats(stats)
    try:
        x = _graded(rng, 4000, 200, 1e10)
        b, flag = _basis(ctx, cuda, x)
        assert stats.tolist()[1] == 1, "expected the Householder hand-over"
    finally:
        ctx.cholqr_stats(None)
    assert flag == 0
    assert np.abs(b.T @ b - np.eye(200)).max() < 1e-13
    r = b.T @ x  # the unique QR: B orthonormal, BᵀX upper triangular with a positive diagonal, B·R = X
    assert np.abs(np.tril(r, -1)).max() < 1e-13 * np.abs(r).max()
    assert np.all(np.diag(r) > 0)
    assert np.abs(b @ r - x).max() < 1e-13 * np.abs(x).max()


@pytest.mark.parametrize("kappa", [1e8, 1e11])
def test_shifted_route_as_a_basis(cuda, kappa):
    """n ≥ 384 beyond the Cholesky guard: the shifted route runs, and as a basis
    it may stop after its second pass (κ₂(Q₁) small, decided on the device from
    R₂: κ = 1e8 here) or run all three (κ = 1e11).  Either way B = Q·T with T
    upper triangular near I, and qr(B) returns Q."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(14)
    x = _graded(rng, 3000, 400, kappa)
    stats = torch.zeros(4, dtype=torch.int32, device=cuda)
    ctx.cholqr_stats(stats)
    try:
        b, flag = _basis(ctx, cuda, x)
        st = stats.tolist()
    finally:
        ctx.cholqr_stats(None)
    assert flag == 0
    assert st[0] == 1 and st[1] == 0 and st[3] == 1, st  # completed by the shifted route, no Householder hand-over
    defect = np.abs(b.T @ b - np.eye(400)).max()
    assert defect < (1e-4 if kappa < 1e10 else 1e-13), defect
    q, r = oracle_qr(x)
    qb, _ = oracle_qr(b)
    tol = conditioning_tolerance(r.T, strict=1e-10)
    assert np.all(column_relative_error(qb, q) <= tol)


def test_looser_guard_for_a_basis(cuda):
    """κ₂ = 5e5 (κ₁, the guard's 1-norm estimate, runs ~10× higher) fails the
    full QR's κ₁ ≤ 1e6 guard but stays on the one-pass route as a basis
    (CQ_KAPPA_MAX_BASIS): B = Q·T with T within 1e-2 of I."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(8)
    x = _graded(rng, 6000, 200, 5e5)
    stats = torch.zeros(4, dtype=torch.int32, device=cuda)
    ctx.cholqr_stats(stats)
    try:
        b, flag = _basis(ctx, cuda, x)
        assert stats.tolist()[:2] == [1, 0], "expected the one-pass route, no hand-over"
        stats.zero_()
        full = _dev_matrix(x, cuda)
        D.householder_qr_(ctx, full)
        torch.cuda.synchronize()
        assert stats.tolist()[1] == 1, "the full QR of the same input should leave the Cholesky route"
    finally:
        ctx.cholqr_stats(None)
    assert flag == 0
    q, r = oracle_qr(x)
    t = q.T @ b
    assert np.abs(t.T @ t - np.eye(200)).max() < 1e-2
    assert np.all(np.diag(t) > 0.9)
    # range(B) = range(X) to the accuracy of any QR of X: the component of B outside range(Q) is ~ u·κ₂
    assert np.abs(b - q @ t).max() < 1e-8
    qb, _ = oracle_qr(b)
    tol = conditioning_tolerance(r.T, strict=1e-10)
    assert np.all(column_relative_error(qb, q) <= tol)


def test_rank_flags(cuda):
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(5)
    low = rng.standard_normal((4000, 3)) @ rng.standard_normal((3, 200))
    for x, expect in ((low, 1), (np.zeros((4000, 200)), 2), (rng.standard_normal((4000, 200)), 0)):
        _, flag = _basis(ctx, cuda, x)
        assert flag == expect


def test_switch_off_returns_q(cuda):
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(6)
    x = rng.standard_normal((4000, 200))
    ctx.set_basis_orth(False)
    try:
        b, _ = _basis(ctx, cuda, x)
    finally:
        ctx.set_basis_orth(True)
    q, _ = oracle_qr(x)
    assert np.abs(b.T @ b - np.eye(200)).max() < 1e-13
    assert column_relative_error(b, q).max() < 1e-11


@pytest.mark.parametrize("q", [1, 2, 3])
@pytest.mark.parametrize("shape,d", [((3000, 2500), 160), ((12000, 1500), 64), ((1500, 2500), 500)])
def test_pipeline_unchanged_by_the_switch(cuda, shape, d, q):
    """pbp_qlp with basis-only intermediate orths against the oracle, and against
    itself with every orth run in full: the factors agree far inside the parity
    tolerance, the warnings and the orth count are the same."""
    from paper_2103_07245_b200 import clear_plan_cache, pbp_qlp
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(shape[0] + d + q)
    r = 2 * d
    a = (rng.standard_normal((shape[0], r)) * np.logspace(0, -6, r)) @ rng.standard_normal((r, shape[1]))
    a += 1e-8 * rng.standard_normal(shape)
    got = pbp_qlp(a, d, q=q, seed=7)
    ctx.set_basis_orth(False)
    clear_plan_cache()
    try:
        full = pbp_qlp(a, d, q=q, seed=7)
    finally:
        ctx.set_basis_orth(True)
        clear_plan_cache()
    ref = oracle_pbp_qlp(a, d, q=q, seed=7)
    tol = conditioning_tolerance(ref["l"], strict=1e-10)
    for name, x, f, o in (("Q", got.q_basis, full.q_basis, ref["q"]), ("P", got.p_basis, full.p_basis, ref["p"])):
        assert np.all(column_relative_error(x, o) <= tol), name
        assert np.all(column_relative_error(x, f) <= tol), name
    lref = np.abs(np.diag(ref["l"]))
    assert np.max(np.abs(np.abs(np.diag(got.l)) - lref) / lref) < 1e-10
    assert np.max(np.abs(np.abs(np.diag(got.l)) - np.abs(np.diag(full.l))) / lref) < 1e-10
