"""Parity of the individual sm_100a kernels behind the C ABI.

GEMMs are checked against an exact-enough FP64 reference (numpy dgemm on the
host), the QR against the oracle's LAPACK path (reference linalg.py:106-115),
and the sketch against numpy's own Generator (linalg.py:83-93).
"""
import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import c_gaussian, column_relative_error, oracle_gaussian, oracle_qr, rank_flag

pytestmark = pytest.mark.gpu


def _dev_matrix(x, dev):
    from paper_2103_07245_b200 import device as D

    t = D.empty_matrix(x.shape[0], x.shape[1], dev)
    t.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return t


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (130, 40, 1000), (1000, 40, 1000), (257, 100, 4001),
                                   (512, 256, 2048), (10000, 256, 300), (300, 129, 77)])
@pytest.mark.parametrize("trans", [True, False])
def test_gemm_matches_fp64(cuda, M, N, K, trans):
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(M * 7 + N * 3 + K)
    a = rng.standard_normal((K, M) if trans else (M, K))
    b = rng.standard_normal((K, N))
    ref = (a.T if trans else a) @ b
    ctx = D.context(cuda)
    out = D.gemm(ctx, _dev_matrix(a, cuda), _dev_matrix(b, cuda), trans_a=trans)
    got = out.cpu().numpy()
    # FP64 summation-order difference bound: ~K·u·Σ|a||b|
    bound = 4 * K * 2.0**-53 * ((np.abs(a.T if trans else a)) @ np.abs(b))
    assert np.all(np.abs(got - ref) <= bound + 1e-300)


def test_gemm_alpha_beta_and_determinism(cuda):
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(5)
    a = rng.standard_normal((3000, 700))
    b = rng.standard_normal((3000, 130))
    c0 = rng.standard_normal((700, 130))
    ctx = D.context(cuda)
    A, B = _dev_matrix(a, cuda), _dev_matrix(b, cuda)
    C = _dev_matrix(c0, cuda)
    D.gemm(ctx, A, B, trans_a=True, out=C, alpha=-0.5, beta=2.0)
    ref = -0.5 * a.T @ b + 2.0 * c0
    assert np.abs(C.cpu().numpy() - ref).max() < 1e-10
    r1 = D.gemm(ctx, A, B, trans_a=True).cpu().numpy()
    r2 = D.gemm(ctx, A, B, trans_a=True).cpu().numpy()
    assert np.array_equal(r1, r2)  # stream-K fix-up order is fixed


@pytest.mark.gpu
def test_gemm_concurrent_streams_one_context(cuda):
    """Stream-K GEMMs of ONE context on several streams at once (each call
    with its own workspace, include/pbq.h): every stream has its own flag
    array, so the fix-ups cannot consume each other's partials."""
    import torch

    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(17)
    ctx = D.context(cuda)
    mats = [(rng.standard_normal((4100, 900 + 64 * i)), rng.standard_normal((4100, 200))) for i in range(4)]
    devs = [(_dev_matrix(a, cuda), _dev_matrix(b, cuda)) for a, b in mats]
    serial = [D.gemm(ctx, A, B, trans_a=True).cpu().numpy() for A, B in devs]
    streams = [torch.cuda.Stream(cuda) for _ in devs]
    for rep in range(3):
        outs = []
        torch.cuda.synchronize()
        for (A, B), s in zip(devs, streams):
            with torch.cuda.stream(s):
                outs.append([D.gemm(ctx, A, B, trans_a=True) for _ in range(4)])
        torch.cuda.synchronize()
        for got, ref in zip(outs, serial):
            for g in got:
                assert np.array_equal(g.cpu().numpy(), ref)


def test_gemm_nonfinite_flag(cuda):
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    a = np.ones((517, 300))
    b = np.ones((517, 40))
    flag = torch.zeros(1, dtype=torch.int32, device=cuda)
    D.gemm(ctx, _dev_matrix(a, cuda), _dev_matrix(b, cuda), trans_a=True, nonfinite=flag)
    assert int(flag.item()) == 0
    a[516, 299] = np.inf
    D.gemm(ctx, _dev_matrix(a, cuda), _dev_matrix(b, cuda), trans_a=True, nonfinite=flag)
    assert int(flag.item()) == 1


@pytest.mark.parametrize("m,n", [(1, 1), (5, 5), (40, 40), (64, 33), (1000, 40), (4000, 100), (10000, 256),
                                 (256, 256), (2500, 301), (700, 1), (3000, 544)])
def test_qr_matches_lapack(cuda, qr_method, m, n):
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(m + 31 * n)
    x = rng.standard_normal((m, n))
    qr, rr = oracle_qr(x)
    ctx = D.context(cuda)
    t = _dev_matrix(x, cuda)
    r = D.empty_matrix(n, n, cuda)
    flag = torch.full((1,), -1, dtype=torch.int32, device=cuda)
    D.householder_qr_(ctx, t, r, want_q=True, rank_flag=flag)
    q = t.cpu().numpy()
    rg = r.cpu().numpy()
    assert int(flag.item()) == rank_flag(rr)
    assert np.all(np.diag(rg) >= 0)
    assert np.array_equal(np.tril(rg, -1), np.zeros((n, n)))
    assert column_relative_error(q, qr).max() < 1e-11
    assert np.abs(rg - rr).max() <= 1e-11 * np.abs(rr).max()
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-13


@pytest.mark.parametrize("m,n,decades", [(30000, 48, 6), (100000, 40, 10), (60000, 100, 8), (200000, 64, 12),
                                         (40000, 33, 9)])
def test_qr_graded_rows_beyond_shared_memory(cuda, qr_method, m, n, decades):
    """Column-graded tall inputs whose per-CTA rows exceed shared memory: the
    Cholesky-QR guard hands them to the Householder kernel, whose panels then
    need the column-by-column fallback on rows streamed from A (regression:
    that combination used to leave the panel unfactored)."""
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(m + n)
    x = rng.standard_normal((m, n)) * np.logspace(0, -decades, n)[rng.permutation(n)]
    qr, rr = oracle_qr(x)
    ctx = D.context(cuda)
    t = _dev_matrix(x, cuda)
    r = D.empty_matrix(n, n, cuda)
    D.householder_qr_(ctx, t, r, want_q=True)
    q, rg = t.cpu().numpy(), r.cpu().numpy()
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-13
    colnorm = np.linalg.norm(x, axis=0)
    assert np.all(np.linalg.norm(q @ rg - x, axis=0) <= 1e-14 * np.sqrt(m) * colnorm)
    assert column_relative_error(q, qr).max() < 1e-10
    d = np.abs(np.diag(rr))
    assert np.all(np.abs(np.diag(rg) - d) <= 1e-12 * d)


def test_qr_rank_deficient_rows_beyond_shared_memory(cuda, qr_method):
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(3)
    x = rng.standard_normal((50000, 3)) @ rng.standard_normal((3, 20))
    ctx = D.context(cuda)
    t = _dev_matrix(x, cuda)
    r = D.empty_matrix(20, 20, cuda)
    flag = torch.full((1,), -1, dtype=torch.int32, device=cuda)
    D.householder_qr_(ctx, t, r, want_q=True, rank_flag=flag)
    q, rg = t.cpu().numpy(), r.cpu().numpy()
    assert int(flag.item()) == 1
    assert np.abs(q.T @ q - np.eye(20)).max() < 1e-13
    assert np.abs(q @ rg - x).max() <= 1e-13 * np.abs(x).max() * 10


def test_qr_rank_flags(cuda, qr_method):
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    rng = np.random.default_rng(1)
    low = rng.standard_normal((300, 3)) @ rng.standard_normal((3, 20))
    for x, expect in ((low, 1), (np.zeros((50, 10)), 2), (rng.standard_normal((80, 10)), 0)):
        t = _dev_matrix(x, cuda)
        flag = torch.full((1,), -1, dtype=torch.int32, device=cuda)
        D.householder_qr_(ctx, t, D.empty_matrix(x.shape[1], x.shape[1], cuda), rank_flag=flag)
        assert int(flag.item()) == expect


def _cholqr_counts(ctx, cuda, x):
    from paper_2103_07245_b200 import device as D

    stats = torch.zeros(4, dtype=torch.int32, device=cuda)
    ctx.cholqr_stats(stats)
    try:
        t = _dev_matrix(x, cuda)
        r = D.empty_matrix(x.shape[1], x.shape[1], cuda)
        flag = torch.full((1,), -1, dtype=torch.int32, device=cuda)
        D.householder_qr_(ctx, t, r, rank_flag=flag)
        return stats.tolist(), t.cpu().numpy(), r.cpu().numpy(), int(flag.item())
    finally:
        ctx.cholqr_stats(None)


def test_shifted_cholqr3_route(cuda):
    """n ≥ 384: an input that fails the κ₁ guard goes through the shifted
    Cholesky-QR3 route (still GEMM-shaped passes) instead of the Householder
    kernel; only an exactly singular one reaches Householder."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    ctx.set_qr_method(ctx.QR_AUTO)
    rng = np.random.default_rng(11)
    for m, n, logk in ((4000, 400, 10), (512, 512, 9), (3000, 416, 12)):
        u, _ = np.linalg.qr(rng.standard_normal((m, n)))
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        x = (u * np.logspace(0, -logk, n)) @ v.T
        counts, q, r, flag = _cholqr_counts(ctx, cuda, x)
        assert counts == [1, 0, counts[2], 1], (m, n, counts)
        qr_, rr = oracle_qr(x)
        assert flag == rank_flag(rr) == 0
        kj = np.abs(rr[0, 0]) / np.abs(np.diag(rr))
        tol = np.maximum(1e-10, 64 * 2.0**-53 * kj)
        assert np.all(column_relative_error(q, qr_) <= tol), (m, n)
        assert np.abs(q.T @ q - np.eye(n)).max() < 1e-12
    # exactly rank deficient: the shifted route's later passes fail → Householder
    b = rng.standard_normal((2000, 400))
    b[:, 200:] = b[:, :200] @ rng.standard_normal((200, 200))
    counts, q, r, flag = _cholqr_counts(ctx, cuda, b)
    assert counts[1] == 1 and counts[0] == 0 and flag == 1


@pytest.mark.parametrize("family", ["auto", "chain"])
def test_cholqr_path_and_guard(cuda, family):
    """The default method completes well-conditioned inputs (κ₁ ≤ 1e6, both
    the series and the Cholesky variant of pass 2) by Cholesky-QR2 and hands
    ill-conditioned, rank-deficient and zero inputs to the Householder kernel
    on the device; either way the factors match LAPACK (linalg.py:106-115).
    "auto" runs n ≤ 128 through the single-launch kernel
    (cholqr_small_f64.cuh), "chain" forces the multi-launch chain."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    ctx.set_qr_method(ctx.QR_AUTO)
    rng = np.random.default_rng(5)
    u, _ = np.linalg.qr(rng.standard_normal((3000, 96)))
    v, _ = np.linalg.qr(rng.standard_normal((96, 96)))
    # expected [done, Householder fallbacks, pass 2 by the near-identity series, done by the shifted route];
    # method 2 forces the blocked Cholesky in pass 2 (its safety path: the κ₁
    # guard fires long before G₂ stops being near the identity)
    cases = [
        ("gaussian", rng.standard_normal((3000, 96)), [1, 0, 1, 0], 0),
        ("graded 1e-4", rng.standard_normal((3000, 96)) * np.logspace(0, -4, 96), [1, 0, 1, 0], 0),
        ("kappa 1e5", (u * np.logspace(0, -5, 96)) @ v.T, [1, 0, 1, 0], 0),
        ("kappa 1e12", (u * np.logspace(0, -12, 96)) @ v.T, [0, 1, 0, 0], 0),
        ("rank deficient", np.hstack([u[:, :40], u[:, :40] @ rng.standard_normal((40, 56))]), [0, 1, 0, 0], 0),
        ("zero", np.zeros((300, 40)), [0, 1, 0, 0], 0),
        ("gaussian, no series", rng.standard_normal((3000, 96)), [1, 0, 0, 0], 2),
        ("kappa 1e5, no series", (u * np.logspace(0, -5, 96)) @ v.T, [1, 0, 0, 0], 2),
        ("300x257, no series", rng.standard_normal((300, 257)), [1, 0, 0, 0], 2),
        # 128 < n ≤ 256 with few rows: the mid-size single launch (cholqr_mid_f64.cuh) under "auto"
        ("mid 400x200", rng.standard_normal((400, 200)), [1, 0, 1, 0], 0),
        ("mid 256x256, no series", rng.standard_normal((256, 256)), [1, 0, 0, 0], 2),
        ("mid kappa 1e12", (np.linalg.qr(rng.standard_normal((400, 160)))[0] * np.logspace(0, -12, 160))
         @ np.linalg.qr(rng.standard_normal((160, 160)))[0].T, [0, 1, 0, 0], 0),
    ]
    for name, x, expect, method in cases:
        if family == "chain" and method == 0:
            method = ctx.QR_CHOLQR_CHAIN
        ctx.set_qr_method(method)
        try:
            counts, q, r, flag = _cholqr_counts(ctx, cuda, x)
        finally:
            ctx.set_qr_method(ctx.QR_AUTO)
        assert counts == expect, (name, counts)
        qr_, rr = oracle_qr(x)
        assert flag == rank_flag(rr), name
        if rank_flag(rr) == 0:
            kappa = np.linalg.cond(x)
            tol = max(1e-11, 64 * 2.0**-53 * kappa)
            assert column_relative_error(q, qr_).max() < tol, name
            assert np.abs(q.T @ q - np.eye(x.shape[1])).max() < 1e-13, name
        assert np.abs(r - rr).max() <= 1e-11 * max(np.abs(rr).max(), 1e-300), name


@pytest.mark.parametrize("rows,cols,seed", [(1, 1, 0), (7, 13, 2**100 + 7), (1000, 40, 0), (4000, 100, 1),
                                            (20000, 256, 12345)])
def test_gaussian_matches_numpy(cuda, rows, cols, seed):
    from paper_2103_07245_b200 import gaussian_matrix

    got = gaussian_matrix(rows, cols, seed)
    ref = oracle_gaussian(rows, cols, seed)
    # bit-exact, exponential-tail draws included (glibc_log1p, sketch.cuh)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("seed", [0, 7, 2**64 + 5])
def test_gaussian_bitwise_many_tail_draws(cuda, seed):
    """4 M normals (≈ 1000 exponential-tail draws, ≈ 4e4 wedge tests) per
    seed: every value bitwise numpy's, the tails included."""
    from paper_2103_07245_b200 import gaussian_matrix

    got = gaussian_matrix(4000, 1000, seed)
    ref = oracle_gaussian(4000, 1000, seed)
    assert np.count_nonzero(np.abs(ref) > 3.6541528853610088) > 500  # the tail branch was exercised
    assert np.array_equal(got, ref)


def test_gaussian_row_offset(cuda):
    from paper_2103_07245_b200 import gaussian_matrix

    full = gaussian_matrix(3000, 64, 9)
    part = gaussian_matrix(1000, 64, 9, row_offset=1500)
    assert np.array_equal(part, full[1500:2500])
    ref = c_gaussian(1000, 64, 9, row_offset=1500)
    assert np.array_equal(part, ref)
    # a block deep in the stream: the prefix chunks are walked for the chain
    # only (no value write-out), the block itself is bitwise numpy's
    deep = gaussian_matrix(300, 37, 2**70 + 3, row_offset=40000)
    assert np.array_equal(deep, oracle_gaussian(40300, 37, 2**70 + 3)[40000:])
    assert np.array_equal(gaussian_matrix(1, 5, 4, row_offset=7), oracle_gaussian(8, 5, 4)[7:])


@pytest.mark.parametrize("n1,n2,d,rank", [(300, 200, 25, None), (301, 257, 33, 7), (1000, 40, 40, 40),
                                          (2000, 1500, 100, 64), (129, 65, 65, 1)])
def test_residual_norms_match_numpy(cuda, n1, n2, d, rank):
    """Fused one-pass ‖A − Q_k L_k P_kᵀ‖_F vs the dense numpy
    residual of QlpFactors.approx(rank) (algorithms.py:101-106)."""
    from paper_2103_07245_b200 import pbp_qlp, reconstruction_error, residual_norms

    rng = np.random.default_rng(n1 + n2 + d)
    a = rng.standard_normal((n1, d)) @ rng.standard_normal((d, n2)) / d + 1e-2 * rng.standard_normal((n1, n2))
    f = pbp_qlp(a, d, q=1, seed=3)
    r, na = residual_norms(a, f, rank)
    k = d if rank is None else rank
    ref = np.linalg.norm(a - f.q_basis[:, :k] @ f.l[:k, :k] @ f.p_basis[:, :k].T)
    assert abs(r - ref) <= 1e-12 * np.linalg.norm(a) + 1e-10 * ref
    assert abs(na - np.linalg.norm(a)) <= 1e-13 * np.linalg.norm(a)
    assert abs(reconstruction_error(a, f, rank) - ref / np.linalg.norm(a)) <= 1e-12
    assert abs(f.frobenius_error(a, rank) - ref) <= 1e-12 * np.linalg.norm(a) + 1e-10 * ref
    # deterministic: same bits on a second call
    assert residual_norms(a, f, rank) == (r, na)


@pytest.mark.parametrize("m,n,logk", [(129, 129, 13), (256, 256, 13), (129, 129, 8), (1000, 129, 13), (500, 96, 13)])
def test_householder_orthogonality_ill_conditioned(cuda, m, n, logk):
    """The Householder kernel's Q stays orthonormal to LAPACK's level on
    ill-conditioned inputs (its fast panel path is taken only by panels whose
    min/max diag(R₁) is at least 0.1; below that the reconstructed reflectors
    lost orthogonality: 3.3e-9 at 129×129, κ = 1e13, with the old 1e-4)."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    ctx.set_qr_method(ctx.QR_HOUSEHOLDER)
    try:
        rng = np.random.default_rng(m + n + logk)
        u, _ = np.linalg.qr(rng.standard_normal((m, n)))
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        x = (u * np.logspace(0, -logk, n)) @ v.T
        t = D.as_kernel_operand(torch.from_numpy(x).to(cuda))
        r = D.empty_matrix(n, n, cuda)
        D.householder_qr_(ctx, t, r)
        q = t.cpu().numpy()
    finally:
        ctx.set_qr_method(ctx.QR_AUTO)
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-14
    assert np.abs(q @ r.cpu().numpy() - x).max() < 1e-14 * np.abs(x).max() * n
