"""cor_utv and its column-pivoted QR core on the B200 kernels
against the reference's golden fixtures (tests/golden/make_golden_utv.py),
the live oracle (oracle_cor_utv / oracle_column_pivoted_qr, LAPACK dgeqp3) and
the reference's own test_algorithms.py::TestCompressedUtv and
test_linalg.py::TestColumnPivotedQr properties.

Pivots are compared exactly wherever they are numerically determined: on
inputs with distinct column norms, and on the leading block of a UTV core
whose diagonal stays above the noise floor.  Beyond that block the core is
rounding noise in the reference itself (its pivot order there is decided by
OpenBLAS's per-column rounding), so the tail is checked through
reconstruction and orthonormality instead."""
import json
import os
import warnings

import numpy as np
import pytest

from oracle.pbp_qlp_oracle import (
    column_relative_error,
    cpqr_pivots_restated,
    oracle_column_pivoted_qr,
    oracle_cor_utv,
)
from tests.golden.recipes import CPQR_CASES, UTV_CASES, make_input

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest_utv.json")))
U = 2.0**-53


def _significant(t, rel=1e-9):
    """Length of the leading run of |t_jj| > rel·|t_00| (the determined block)."""
    d = np.abs(np.diag(t))
    if d.size == 0 or d[0] == 0:
        return 0
    ok = d > rel * d[0]
    return int(np.argmin(ok)) if not ok.all() else d.size


def _determined(core, t, gap=1e-10):
    """Pivots are numerically determined up to the first step whose margin
    over the runner-up is at rounding level, and only above the noise floor."""
    _, gaps = cpqr_pivots_restated(core, return_gaps=True)
    close = np.flatnonzero(gaps < gap)
    return min(_significant(t), int(close[0]) if close.size else gaps.size)


def _kappa(rdiag):
    with np.errstate(divide="ignore"):
        return np.where(rdiag > 0, rdiag[0] / rdiag, np.inf) if rdiag.size and rdiag[0] > 0 else np.ones(rdiag.size)


def _check_utv(a, f, ref_u, ref_t, ref_v, ref, strict=1e-10):
    """Determined block: per column max(strict, 64·u·κ_j) with κ_j from the
    core's T and from the orth inputs of V̄ (column perm_j) and Ū (worst
    column) — the non-reorthonormalized branch orthonormalizes A(AᵀA)^q Ω
    once, so its bases are only determined to u·κ of that sample.  On the
    pass-efficient non-reorthonormalized branch the core is pinv(gram)ᵀ·…
    (algorithms.py:295-303): LAPACK's own singular values of gram carry an
    absolute error ~u·σ₀, i.e. a relative u·κ₂(gram) on the smallest kept one,
    so the reference's core itself is determined only to ~u·κ₂(gram)."""
    k = _determined(ref["core"], ref_t)
    if k:
        d = np.abs(np.diag(ref_t))[:k]
        perm = ref["perm"][:k]
        ku = _kappa(ref["rdiag_ubar"])
        kv = _kappa(ref["rdiag_vbar"])
        tol_core = np.maximum(strict, 64 * U * ref.get("pinv_kappa", 1.0) * d[0] / d)
        tol_v = np.maximum(tol_core, 64 * U * kv[perm] * (d[0] / d))
        tol_u = np.maximum(tol_core, 64 * U * ku.max() * (d[0] / d))
        assert np.all(column_relative_error(f.v[:, :k], ref_v[:, :k]) <= tol_v)
        assert np.all(column_relative_error(f.u[:, :k], ref_u[:, :k]) <= tol_u)
        rows = np.linalg.norm(f.t[:k] - ref_t[:k], axis=1) / np.linalg.norm(ref_t[:k], axis=1)
        assert np.all(rows <= np.maximum(tol_u, tol_v))
    # everything: structure, orthonormal bases, reconstruction as good as the reference's
    assert np.array_equal(f.t, np.triu(f.t))
    for b in (f.u, f.v):
        np.testing.assert_allclose(b.T @ b, np.eye(b.shape[1]), atol=1e-11)
    na = np.linalg.norm(a)
    e_got = np.linalg.norm(a - f.u @ f.t @ f.v.T) / na
    e_ref = np.linalg.norm(a - ref_u @ ref_t @ ref_v.T) / na
    assert abs(e_got - e_ref) <= 1e-10
    return k


@pytest.mark.parametrize("name", sorted(UTV_CASES))
def test_cor_utv_matches_golden(cuda, name):
    from paper_2103_07245_b200.utv import cor_utv

    case = MANIFEST["utv"][name]
    a = make_input(UTV_CASES[name]["recipe"])
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        f = cor_utv(a, case["d"], q=case["q"], seed=case["seed"], pass_efficient=case["pass_efficient"],
                    reorthonormalize=case["reorth"])
    assert sum(1 for w in rec if "orth:" in str(w.message)) == case["rank_warnings"]
    assert f.sketch.passes_over_a == case["passes_over_a"]
    assert f.pinv_truncated == case["pinv_truncated"]
    assert f.pass_efficient == case["pass_efficient"]
    assert f.u.shape == g["u"].shape and f.t.shape == g["t"].shape and f.v.shape == g["v"].shape
    ref = oracle_cor_utv(a, case["d"], q=case["q"], seed=case["seed"], pass_efficient=case["pass_efficient"],
                         reorthonormalize=case["reorth"])
    _check_utv(a, f, g["u"], g["t"], g["v"], ref)


@pytest.mark.parametrize("pe,reorth,q", [(False, True, 0), (False, True, 2), (True, True, 1), (True, False, 1),
                                          (False, False, 1)])
def test_cor_utv_matches_oracle_graded(cuda, pe, reorth, q):
    from paper_2103_07245_b200.utv import cor_utv

    rng = np.random.default_rng(5)
    n1, n2, r = 900, 700, 120
    u, _ = np.linalg.qr(rng.standard_normal((n1, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n2, r)))
    a = (u * np.exp(-np.arange(r) / 12.0)) @ v.T + 1e-7 * rng.standard_normal((n1, n2))
    f = cor_utv(a, 64, q=q, seed=11, pass_efficient=pe, reorthonormalize=reorth)
    ref = oracle_cor_utv(a, 64, q=q, seed=11, pass_efficient=pe, reorthonormalize=reorth)
    k = _check_utv(a, f, ref["u"], ref["t"], ref["v"], ref)
    assert k >= 40
    assert f.sketch.passes_over_a == ref["passes"]


def test_reference_properties(cuda):
    """test_algorithms.py:124-156 (TestCompressedUtv) on the device path."""
    from paper_2103_07245_b200.utv import cor_utv

    def planted(rows, cols, values, seed):
        rng = np.random.default_rng(seed)
        u, _ = np.linalg.qr(rng.standard_normal((rows, len(values))))
        v, _ = np.linalg.qr(rng.standard_normal((cols, len(values))))
        return (u * np.asarray(values)) @ v.T

    values = np.linspace(1, 0.1, 10)
    a = planted(50, 40, values, 11)
    f = cor_utv(a, 10, seed=2)
    assert not f.pass_efficient and f.sketch.passes_over_a == 3
    assert np.linalg.norm(a - f.approx(), 2) <= 1e-12
    assert np.allclose(f.t, np.triu(f.t))
    a = planted(100, 80, values, 12)
    for reorth in (True, False):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            f = cor_utv(a, 20, seed=3, pass_efficient=True, reorthonormalize=reorth)
        assert f.pass_efficient and f.sketch.passes_over_a == 2
        assert np.linalg.norm(a - f.approx(), 2) <= 1e-8 * values[0]
    eye = np.eye(4)
    for pe in (False, True):
        assert np.linalg.norm(eye - cor_utv(eye, 4, seed=0, pass_efficient=pe).approx(), 2) <= 1e-12
    a = planted(30, 20, np.array([1.0, 1e-14, 1e-15]), 13)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert cor_utv(a, 6, seed=1, pass_efficient=True, reorthonormalize=False).pinv_truncated


def test_cor_utv_torch_in_torch_out(cuda):
    import torch

    from paper_2103_07245_b200.utv import cor_utv

    a = torch.randn(300, 200, dtype=torch.float64, device=cuda)
    f = cor_utv(a, 16, q=1, seed=3)
    assert isinstance(f.u, torch.Tensor) and f.u.device == a.device
    ref = oracle_cor_utv(a.cpu().numpy(), 16, q=1, seed=3)
    e = torch.linalg.norm(a - f.approx()) / torch.linalg.norm(a)
    e_ref = np.linalg.norm(a.cpu().numpy() - ref["u"] @ ref["t"] @ ref["v"].T) / np.linalg.norm(a.cpu().numpy())
    assert abs(float(e) - e_ref) <= 1e-10


def test_cor_utv_errors(cuda):
    from paper_2103_07245_b200 import exceptions as exc
    from paper_2103_07245_b200.utv import cor_utv

    with pytest.raises(exc.ParameterError):
        cor_utv(np.ones((5, 4)), 5)
    a = np.ones((6, 5))
    a[1, 1] = np.inf
    with pytest.raises(exc.MatrixInputError):
        cor_utv(a, 2)


# ------------------------------------------------------- column_pivoted_qr --
@pytest.mark.parametrize("name", sorted(CPQR_CASES))
def test_cpqr_matches_golden(cuda, name):
    from paper_2103_07245_b200.linalg import column_pivoted_qr

    m = make_input(CPQR_CASES[name])
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    q, r, perm = column_pivoted_qr(m)
    assert perm.dtype == np.int32 and list(perm) == MANIFEST["cpqr"][name]["perm"]
    scale = max(1.0, np.abs(m).max())
    np.testing.assert_allclose(q @ r, m[:, perm], atol=1e-12 * scale)
    np.testing.assert_allclose(r, g["r"], atol=1e-11 * scale)
    assert np.all(np.diag(r) >= 0) and np.array_equal(r, np.triu(r))


@pytest.mark.parametrize("shape,decades", [((300, 200), 10), ((256, 256), 6), ((1024, 1024), 8), ((700, 1500), 5),
                                           ((2000, 64), 12)])
def test_cpqr_pivots_match_lapack(cuda, shape, decades):
    """Distinct norms: the device pivots are LAPACK dgeqp3's, position by position."""
    from paper_2103_07245_b200.linalg import column_pivoted_qr

    rng = np.random.default_rng(sum(shape))
    m = rng.standard_normal(shape) * np.logspace(0, -decades, shape[1])[rng.permutation(shape[1])]
    _, r, perm = column_pivoted_qr(m)
    q0, r0, p0 = oracle_column_pivoted_qr(m)
    assert np.array_equal(perm, p0)
    d = np.abs(np.diag(r0))
    assert np.all(np.abs(np.diag(r) - d) <= 1e-10 * d + 64 * U * d[0])


def test_cpqr_graded_spectrum_core(cuda):
    """A UTV-like core: decaying singular values with random singular vectors."""
    from paper_2103_07245_b200.linalg import column_pivoted_qr

    rng = np.random.default_rng(9)
    n = 512
    m = rng.standard_normal((n, n)) @ np.diag(np.exp(-np.arange(n) / 25)) @ rng.standard_normal((n, n))
    _, r, perm = column_pivoted_qr(m)
    _, r0, p0 = oracle_column_pivoted_qr(m)
    k = min(_significant(r0), _determined(m, r0))
    assert k > 100 and np.array_equal(perm[:k], p0[:k])


def test_cpqr_properties(cuda):
    """test_linalg.py:72-91 (TestColumnPivotedQr) on the device."""
    import torch

    from paper_2103_07245_b200.linalg import column_pivoted_qr

    rng = np.random.default_rng(2)
    m = rng.standard_normal((40, 15))
    q, r, perm = column_pivoted_qr(m)
    assert sorted(perm) == list(range(15))
    np.testing.assert_allclose(q @ r, m[:, perm], atol=1e-12 * np.linalg.norm(m, 2))
    diag = np.abs(np.diag(column_pivoted_qr(np.random.default_rng(9).standard_normal((60, 25)))[1]))
    assert np.all(diag[:-1] >= diag[1:] - 1e-14)
    m = np.random.default_rng(4).standard_normal((30, 10)) * np.logspace(0, -8, 10)
    assert column_pivoted_qr(m)[2][0] == int(np.argmax(np.linalg.norm(m, axis=0)))
    t = torch.from_numpy(m).to(cuda)
    qt, rt, pt = column_pivoted_qr(t)
    assert pt.device == t.device and torch.equal(pt.cpu(), torch.from_numpy(column_pivoted_qr(m)[2]).long())


def test_cpqr_c_abi_direct(cuda):
    """pbq_cpqr_pivots + pbq_gather_columns through ctypes, no Python wrapper."""
    import ctypes

    import torch

    from paper_2103_07245_b200 import _lib
    from paper_2103_07245_b200 import device as dev

    lib = _lib.load()
    ctx = dev.context(cuda)
    rng = np.random.default_rng(3)
    m_host = rng.standard_normal((64, 33)) * np.logspace(0, -5, 33)
    m = dev.as_kernel_operand(torch.from_numpy(m_host).to(cuda))
    perm = torch.empty(33, dtype=torch.int64, device=cuda)
    nb = ctypes.c_size_t()
    assert lib.pbq_cpqr_workspace_bytes(ctx.handle, 64, 33, ctypes.byref(nb)) == 0
    ws = torch.empty(nb.value, dtype=torch.uint8, device=cuda)
    st = lib.pbq_cpqr_pivots(ctx.handle, 64, 33, dev.ptr(m), dev.ld_of(m), dev.ptr(perm), dev.ptr(ws), nb.value,
                             dev.stream_ptr(cuda))
    assert st == 0
    assert np.array_equal(perm.cpu().numpy(), oracle_column_pivoted_qr(m_host)[2])
    out = dev.empty_matrix(64, 33, cuda)
    assert lib.pbq_gather_columns(ctx.handle, 64, 33, dev.ptr(m), dev.ld_of(m), dev.ptr(perm), dev.ptr(out),
                                  dev.ld_of(out), dev.stream_ptr(cuda)) == 0
    assert np.array_equal(out.cpu().numpy(), m_host[:, perm.cpu().numpy()])
    # too small a workspace is refused, not run
    assert lib.pbq_cpqr_pivots(ctx.handle, 64, 33, dev.ptr(m), dev.ld_of(m), dev.ptr(perm), dev.ptr(ws), 16,
                               dev.stream_ptr(cuda)) == _lib.PBQ_ERR_PARAM


def test_cpqr_beyond_shared_memory(cuda):
    """8·m + 8·n past the 227 KB opt-in: the per-CTA vectors move to global scratch."""
    from paper_2103_07245_b200.linalg import column_pivoted_qr

    rng = np.random.default_rng(4)
    m = rng.standard_normal((30000, 48)) * np.logspace(0, -6, 48)[rng.permutation(48)]
    q, r, perm = column_pivoted_qr(m)
    assert np.array_equal(perm, oracle_column_pivoted_qr(m)[2])
    np.testing.assert_allclose(q @ r, m[:, perm], atol=1e-12 * np.abs(m).max())


# ------------------------------------------------------------------ callers --
def test_callers_dispatch_cor_utv_and_cpqr(cuda):
    """factorize / low_rank_approx / error_curve / CorUtv (analysis.py:135-247,
    estimators.py:128-157) on the GPU path."""
    from paper_2103_07245_b200 import analysis
    from paper_2103_07245_b200.estimators import CorUtv
    from oracle.pbp_qlp_oracle import oracle_spectral_norm

    rng = np.random.default_rng(6)
    u, _ = np.linalg.qr(rng.standard_normal((200, 30)))
    v, _ = np.linalg.qr(rng.standard_normal((150, 30)))
    a = (u * 0.8 ** np.arange(30)) @ v.T
    f = analysis.factorize(a, "cor_utv", 12, q=1, seed=2)
    ref = oracle_cor_utv(a, 12, q=1, seed=2)
    np.testing.assert_allclose(analysis.low_rank_approx(f), ref["u"] @ ref["t"] @ ref["v"].T, atol=1e-12)
    np.testing.assert_allclose(analysis.low_rank_approx(f, rank=5),
                               ref["u"][:, :5] @ ref["t"][:5, :5] @ ref["v"][:, :5].T, atol=1e-12)
    c = analysis.factorize(a, "cpqr", 10)
    q0, r0, p0 = oracle_column_pivoted_qr(a)
    k = _determined(a, r0)  # rank 30: the pivots past it are rounding noise
    assert k >= 25 and np.array_equal(c.perm[:k], p0[:k])
    approx = np.empty_like(a)
    approx[:, p0] = q0[:, :7] @ r0[:7, :]
    np.testing.assert_allclose(analysis.low_rank_approx(c, rank=7), approx, atol=1e-12)
    for alg in ("cor_utv", "cpqr"):
        recs = analysis.error_curve(a, alg, [5, 12], q=1, seed=2)
        for rec in recs:
            if alg == "cpqr":
                res = a.copy()
                res[:, p0] -= q0[:, :rec["d"]] @ r0[:rec["d"], :]
                res = -res
            else:
                o = oracle_cor_utv(a, rec["d"], q=1, seed=2)
                res = a - o["u"] @ o["t"] @ o["v"].T
            assert abs(rec["frobenius_error"] - np.linalg.norm(res)) <= 1e-10 * np.linalg.norm(a)
            assert abs(rec["spectral_error"] - oracle_spectral_norm(res)) <= 1e-10 * np.linalg.norm(a, 2)
    est = CorUtv(8, q=1, seed=3).fit(a)
    ref = oracle_cor_utv(a, 8, q=1, seed=3)
    np.testing.assert_allclose(est.components_, ref["v"][:, :8].T, atol=1e-11)
    np.testing.assert_allclose(est.singular_values_, np.abs(np.diag(ref["t"]))[:8], rtol=1e-11)
    z = est.transform(a)
    np.testing.assert_allclose(z, a @ ref["v"][:, :8], atol=1e-11)


def test_integration_installs_cor_utv(cuda, reference_pkg):
    """install() rebinds cor_utv / column_pivoted_qr in the reference (only
    where the reference is importable, i.e. never on the GPU box)."""
    from paper_2103_07245_b200 import integration

    saved = integration.install(reference_pkg)
    try:
        a = np.random.default_rng(1).standard_normal((80, 60))
        f = reference_pkg.cor_utv(a, 10, q=1, seed=4)
        assert isinstance(f, reference_pkg.UtvFactors) and f.sketch.passes_over_a == 5
        c = reference_pkg.column_pivoted_qr(a)
        assert isinstance(c, reference_pkg.QrFactors)
        assert reference_pkg.analysis.factorize(a, "cor_utv", 10, q=1, seed=4).t.shape == (10, 10)
    finally:
        integration.uninstall(saved)


@pytest.mark.parametrize("shape,decades", [((300, 200), 10), ((256, 256), 6), ((90, 40), 4), ((12, 30), 3),
                                           ((640, 600), 7)])
def test_cpqr_cluster_and_grid_kernels_agree(cuda, monkeypatch, shape, decades):
    """The single-cluster kernel (DSMEM, n ≤ ~640) and the cooperative-grid
    kernel implement the same rule: identical pivots, both equal to LAPACK's."""
    import torch

    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    m = rng.standard_normal(shape) * np.logspace(0, -decades, shape[1])[rng.permutation(shape[1])]
    t = D.as_kernel_operand(torch.from_numpy(m).to(cuda))
    ctx = D.context(cuda)
    p_cluster = D.cpqr_pivots(ctx, t).cpu().numpy()
    monkeypatch.setenv("PBQ_CPQR_NO_CLUSTER", "1")
    p_grid = D.cpqr_pivots(ctx, t).cpu().numpy()
    assert np.array_equal(p_cluster, p_grid)
    assert np.array_equal(p_cluster, oracle_column_pivoted_qr(m)[2])
