"""Randomized SVD on the B200 kernels against the oracle
restatement of the reference (algorithms.py:263-292) and the reference's own
test_algorithms.py::TestRandomizedSvd properties.  Singular vectors are
compared up to the joint (u_j, v_j) sign LAPACK leaves free, on spectra whose
singular values are separated (so the vectors are determined)."""
import warnings

import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import column_relative_error, oracle_r_svd

pytestmark = pytest.mark.gpu


def _graded(n1, n2, rank, ratio, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((n1, rank)))
    v, _ = np.linalg.qr(rng.standard_normal((n2, rank)))
    a = (u * ratio ** np.arange(rank)) @ v.T
    return a + noise * rng.standard_normal((n1, n2)) if noise else a


def _check(a, d, q, seed, reorth=True, kcheck=None, tol=1e-10):
    from paper_2103_07245_b200.rsvd import r_svd

    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        f = r_svd(a, d, q=q, seed=seed, reorthonormalize=reorth)
    ref = oracle_r_svd(a, d, q=q, seed=seed, reorthonormalize=reorth)
    assert sum(1 for w in rec if "orth:" in str(w.message)) == sum(1 for x in ref["rank_flags"] if x)
    k = ref["s"].size if kcheck is None else kcheck
    s_tol = np.maximum(tol, 16 * 2.0**-53 * ref["s"][0] / ref["s"][:k])
    assert np.all(np.abs(f.s[:k] - ref["s"][:k]) / ref["s"][:k] <= s_tol)
    # joint sign per column, then column errors
    sgn = np.sign(np.sum(f.u[:, :k] * ref["u"][:, :k], axis=0))
    assert np.all(column_relative_error(f.u[:, :k] * sgn, ref["u"][:, :k]) <= 64 * s_tol)
    assert np.all(column_relative_error(f.v[:, :k] * sgn, ref["v"][:, :k]) <= 64 * s_tol)
    om, ro = f.sketch.test_matrix, ref["omega"]
    assert np.array_equal(om, ro)  # bit-exact device sketch
    assert f.sketch.passes_over_a == 2 * q + 2
    return f, ref


@pytest.mark.parametrize("q,reorth", [(0, True), (1, True), (2, True), (1, False)])
def test_graded_spectrum_matches_oracle(cuda, q, reorth):
    a = _graded(600, 400, 60, 0.85, 1, noise=1e-6)
    _check(a, 30, q, 7, reorth, kcheck=20 if not reorth else None)


def test_reference_properties(cuda):
    """test_algorithms.py:103-124: exact-rank recovery, passes, reorth=False at q=0."""
    from paper_2103_07245_b200.rsvd import r_svd

    rng = np.random.default_rng(0)
    a = rng.standard_normal((50, 12)) @ rng.standard_normal((12, 40))
    f = r_svd(a, 12, seed=1)
    assert np.linalg.norm(a - f.approx()) <= 1e-10 * np.linalg.norm(a)
    assert np.allclose(f.s, np.linalg.svd(a, compute_uv=False)[:12], rtol=1e-10)
    assert r_svd(a, 6, q=2, seed=0).sketch.passes_over_a == 6
    f1 = r_svd(a, 8, q=0, seed=1, reorthonormalize=True)
    f2 = r_svd(a, 8, q=0, seed=1, reorthonormalize=False)
    assert np.allclose(f1.s, f2.s, rtol=1e-12)


def test_wide_d_larger_than_n1(cuda):
    """d ≤ n2 may exceed n1 (algorithms.py:276): orth of the n1×d sample keeps n1 columns."""
    a = _graded(20, 90, 20, 0.7, 3)
    f, ref = _check(a, 40, 1, 2)
    assert f.u.shape == (20, 20) and f.v.shape == (90, 20) and f.s.shape == (20,)


def test_errors_and_device_tensors(cuda):
    from paper_2103_07245_b200 import MatrixInputError, ParameterError
    from paper_2103_07245_b200.rsvd import r_svd

    a = _graded(100, 80, 20, 0.8, 4)
    with pytest.raises(ParameterError, match="d must be in"):
        r_svd(a, 81)
    bad = a.copy()
    bad[3, 4] = np.inf
    with pytest.raises(MatrixInputError):
        r_svd(bad, 10)
    ft = r_svd(torch.from_numpy(a).to(cuda), 10, q=1, seed=5)
    fn = r_svd(a, 10, q=1, seed=5)
    assert ft.u.is_cuda and np.array_equal(ft.s.cpu().numpy(), fn.s)


def test_config3_scale(cuda):
    """BASELINE config-3 shape with r_svd's d = 256, q = 1: the 200 signal
    singular values are separated; the noise ones are not (compare 200)."""
    from paper_2103_07245_b200 import workloads

    a_dev = workloads.make_cfg3(0, cuda)
    a = a_dev.cpu().numpy()
    _check(a, 256, 1, 0, kcheck=150)
