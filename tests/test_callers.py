"""The callers of the path: the `factorize` dispatcher,
`error_curve`, `spectral_norm` and the sklearn `PbpQlp` transformer, against
the reference's own test_estimators.py / test_analysis.py properties and the
oracle.  CPU tests cover argument handling that never reaches the GPU."""
import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import oracle_error_curve, oracle_pbp_qlp, oracle_qr, oracle_spectral_norm


def exact_rank_matrix(rows, cols, rank, seed):
    """test_estimators.py:29-33 (orth = the reference's sign-fixed QR)."""
    rng = np.random.default_rng(seed)
    u = oracle_qr(rng.standard_normal((rows, rank)))[0]
    v = oracle_qr(rng.standard_normal((cols, rank)))[0]
    return (u * np.geomspace(1, 0.1, rank)) @ v.T


# ------------------------------------------------------------------ CPU ----
def test_estimator_params_and_unfitted():
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError

    from paper_2103_07245_b200.estimators import PbpQlp

    est = PbpQlp(n_components=8, q=1, seed=3)
    assert est.get_params() == {"n_components": 8, "q": 1, "seed": 3, "reorthonormalize": True}
    est.set_params(q=2)
    assert clone(est).get_params()["q"] == 2
    with pytest.raises(NotFittedError):
        est.transform(np.ones((3, 4)))


def test_factorize_rejects_other_algorithms_after_validating_a():
    from paper_2103_07245_b200 import MatrixInputError, ParameterError
    from paper_2103_07245_b200.analysis import factorize

    a = np.ones((5, 4))
    with pytest.raises(ParameterError, match="unknown algorithm"):
        factorize(a, "nope", 2)
    with pytest.raises(ParameterError, match="outside the B200 path"):
        factorize(a, "pqlp", 2)
    bad = a.copy()
    bad[0, 0] = np.nan
    with pytest.raises(MatrixInputError):  # analysis.py:140: check_matrix runs before the dispatch
        factorize(bad, "nope", 2)


def test_oracle_spectral_norm_matches_svd():
    rng = np.random.default_rng(0)
    m = rng.standard_normal((2100, 30)) * np.geomspace(1, 1e-2, 30)
    assert abs(oracle_spectral_norm(m) - np.linalg.svd(m, compute_uv=False)[0]) <= 1e-9 * np.linalg.norm(m, 2)


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
class TestPbpQlpEstimator:
    """test_estimators.py:36-119 for PbpQlp, on the GPU path."""

    def _est(self):
        from paper_2103_07245_b200.estimators import PbpQlp

        return PbpQlp(n_components=8, q=1, seed=0)


    def test_fit_transform_shapes(self, cuda):
        x = exact_rank_matrix(40, 30, 8, seed=0)
        est = self._est()
        coords = est.fit_transform(x)
        assert coords.shape == (40, 8)
        assert est.components_.shape == (8, 30)
        assert est.singular_values_.shape == (8,)
        assert est.n_features_in_ == 30

    def test_round_trip_and_parity(self, cuda):
        x = exact_rank_matrix(40, 30, 8, seed=1)
        est = self._est().fit(x)
        rec = est.inverse_transform(est.transform(x))
        assert np.linalg.norm(x - rec, 2) <= 1e-9 * np.linalg.norm(x, 2)
        # the transform is X·componentsᵀ with components from the oracle's P
        ref = oracle_pbp_qlp(x, 8, q=1, seed=0)
        comp = ref["p"][:, :8].T
        s = np.sign(np.sum(est.components_ * comp, axis=1))
        assert np.abs(est.components_ * s[:, None] - comp).max() < 1e-12
        assert np.abs(est.transform(x) * s - x @ comp.T).max() < 1e-12

    def test_components_rows_orthonormal(self, cuda):
        est = self._est().fit(exact_rank_matrix(40, 30, 8, seed=2))
        np.testing.assert_allclose(est.components_ @ est.components_.T, np.eye(8), atol=1e-10)

    def test_singular_values_track_spectrum(self, cuda):
        x = exact_rank_matrix(40, 30, 8, seed=3)
        est = self._est().fit(x)
        assert np.all(est.singular_values_ > 0)
        np.testing.assert_allclose(est.singular_values_, np.abs(np.diag(oracle_pbp_qlp(x, 8, q=1, seed=0)["l"])),
                                   rtol=1e-10)

    def test_column_mismatch_and_excessive_rank(self, cuda):
        from paper_2103_07245_b200 import DimensionError, ParameterError
        from paper_2103_07245_b200.estimators import PbpQlp

        est = self._est().fit(exact_rank_matrix(40, 30, 8, seed=4))
        with pytest.raises(DimensionError):
            est.transform(np.ones((5, 29)))
        with pytest.raises(DimensionError):
            est.inverse_transform(np.ones((5, 7)))
        with pytest.raises(ParameterError):
            PbpQlp(n_components=31).fit(np.ones((40, 30)))

    def test_seed_and_device_tensors(self, cuda):
        from paper_2103_07245_b200.estimators import PbpQlp

        x = exact_rank_matrix(60, 40, 8, seed=5) + 1e-3 * np.random.default_rng(5).standard_normal((60, 40))
        a = PbpQlp(8, seed=1).fit(x).components_
        b = PbpQlp(8, seed=1).fit(x).components_
        assert np.array_equal(a, b)
        xt = torch.from_numpy(x).to(cuda)
        est = PbpQlp(8, seed=1).fit(xt)
        coords = est.transform(xt)
        assert coords.is_cuda and coords.shape == (60, 8)
        assert np.abs(coords.cpu().numpy() - x @ a.T).max() < 1e-12


@pytest.mark.gpu
def test_factorize_is_pbp_qlp(cuda):
    from paper_2103_07245_b200 import pbp_qlp
    from paper_2103_07245_b200.analysis import factorize, low_rank_approx

    rng = np.random.default_rng(7)
    a = rng.standard_normal((200, 120))
    f1 = factorize(a, "pbp_qlp", 20, q=1, seed=4)
    f2 = pbp_qlp(a, 20, q=1, seed=4)
    assert np.array_equal(f1.q_basis, f2.q_basis) and np.array_equal(f1.l, f2.l)
    assert np.allclose(low_rank_approx(f1, 5), f1.q_basis[:, :5] @ f1.l[:5, :5] @ f1.p_basis[:, :5].T)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,d_values,q", [((300, 200), [5, 20, 40], 0), ((2500, 300), [10, 60], 1)])
def test_error_curve_matches_oracle(cuda, shape, d_values, q):
    """analysis.py:213-247: both error kinds per d; (2500, 300) takes the
    power-iteration branch of spectral_norm (max dim > 2000)."""
    from paper_2103_07245_b200.analysis import error_curve

    rng = np.random.default_rng(sum(shape))
    n1, n2 = shape
    a = (rng.standard_normal((n1, 30)) * np.geomspace(1, 1e-2, 30)) @ rng.standard_normal((30, n2)) \
        + 1e-4 * rng.standard_normal((n1, n2))
    got = error_curve(a, "pbp_qlp", d_values, q=q, seed=2)
    ref = oracle_error_curve(a, d_values, q=q, seed=2)
    for g, r in zip(got, ref):
        assert g["d"] == r["d"]
        assert abs(g["frobenius_error"] - r["frobenius_error"]) <= 1e-10 * r["frobenius_error"]
        assert abs(g["spectral_error"] - r["spectral_error"]) <= 1e-8 * r["spectral_error"]


@pytest.mark.gpu
def test_error_curve_r_svd(cuda):
    """error_curve(a, "r_svd", …): frobenius / spectral error of u·diag(s)·vᵀ."""
    from oracle.pbp_qlp_oracle import oracle_r_svd, oracle_spectral_norm
    from paper_2103_07245_b200.analysis import error_curve

    rng = np.random.default_rng(9)
    a = (rng.standard_normal((400, 25)) * np.geomspace(1, 1e-3, 25)) @ rng.standard_normal((25, 250)) \
        + 1e-5 * rng.standard_normal((400, 250))
    for rec in error_curve(a, "r_svd", [8, 20], q=1, seed=3):
        f = oracle_r_svd(a, rec["d"], q=1, seed=3)
        res = a - (f["u"] * f["s"]) @ f["v"].T
        assert abs(rec["frobenius_error"] - np.linalg.norm(res)) <= 1e-9 * np.linalg.norm(res)
        assert abs(rec["spectral_error"] - oracle_spectral_norm(res)) <= 1e-8 * oracle_spectral_norm(res)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_randomized_svd_estimator_protocol(cuda, seed):
    """test_estimators.py:36-95 for RandomizedSvd (GPU r_svd): shapes, exact
    round trip, orthonormal components, spectrum = the oracle's s."""
    from oracle.pbp_qlp_oracle import oracle_r_svd
    from paper_2103_07245_b200.estimators import RandomizedSvd

    x = exact_rank_matrix(40, 30, 8, seed=seed)
    est = RandomizedSvd(n_components=8, q=1, seed=0)
    coords = est.fit_transform(x)
    assert coords.shape == (40, 8) and est.components_.shape == (8, 30)
    assert np.linalg.norm(x - est.inverse_transform(coords), 2) <= 1e-9 * np.linalg.norm(x, 2)
    np.testing.assert_allclose(est.components_ @ est.components_.T, np.eye(8), atol=1e-10)
    np.testing.assert_allclose(est.singular_values_, oracle_r_svd(x, 8, q=1, seed=0)["s"], rtol=1e-10)
