"""Pins the cor_utv / column_pivoted_qr oracle before it is
trusted as the parity checker: against the golden fixtures made by running
the reference (tests/golden/make_golden_utv.py), against the reference itself
when importable, and the dlaqp2 pivot restatement (the rule the device
kernel implements) against scipy's LAPACK dgeqp3."""
import json
import os

import numpy as np
import pytest

from oracle.pbp_qlp_oracle import (
    cpqr_pivots_restated,
    oracle_column_pivoted_qr,
    oracle_cor_utv,
)
from tests.golden.recipes import CPQR_CASES, UTV_CASES, make_input

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest_utv.json")))


def _sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(UTV_CASES))
def test_oracle_cor_utv_matches_golden(name):
    case = MANIFEST["utv"][name]
    a = make_input(UTV_CASES[name]["recipe"])
    assert _sha(a) == case["a_sha256"]
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    o = oracle_cor_utv(a, case["d"], q=case["q"], seed=case["seed"], pass_efficient=case["pass_efficient"],
                       reorthonormalize=case["reorth"])
    assert o["passes"] == case["passes_over_a"]
    assert o["pinv_truncated"] == case["pinv_truncated"]
    assert sum(1 for f in o["rank_flags"] if f) == case["rank_warnings"]
    scale = np.abs(g["t"]).max()
    np.testing.assert_allclose(o["t"], g["t"], rtol=0, atol=1e-12 * scale)
    np.testing.assert_allclose(o["u"] @ o["t"] @ o["v"].T, g["u"] @ g["t"] @ g["v"].T, rtol=0, atol=1e-12 * scale)


@pytest.mark.parametrize("name", sorted(CPQR_CASES))
def test_oracle_cpqr_matches_golden(name):
    case = MANIFEST["cpqr"][name]
    m = make_input(CPQR_CASES[name])
    assert _sha(m) == case["m_sha256"]
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    q, r, perm = oracle_column_pivoted_qr(m)
    assert list(perm) == case["perm"]
    np.testing.assert_allclose(q @ r, m[:, perm], atol=1e-12 * max(1.0, np.abs(m).max()))
    assert np.all(np.diag(r) >= 0)
    np.testing.assert_allclose(r, g["r"], atol=1e-12 * max(1.0, np.abs(m).max()))


@pytest.mark.parametrize("name", sorted(CPQR_CASES))
def test_restated_pivot_rule_matches_lapack_golden(name):
    """dlaqp2 restated (no LAPACK) picks the reference's pivots."""
    assert list(cpqr_pivots_restated(make_input(CPQR_CASES[name]))) == MANIFEST["cpqr"][name]["perm"]


def test_restated_pivot_rule_matches_lapack_random():
    rng = np.random.default_rng(0)
    for _ in range(120):
        m, n = rng.integers(1, 70, 2)
        a = rng.standard_normal((m, n)) * np.logspace(0, rng.uniform(0, 12), n)[rng.permutation(n)]
        assert np.array_equal(cpqr_pivots_restated(a), oracle_column_pivoted_qr(a)[2])
    for n in (128, 200):  # dgeqp3's blocked dlaqps path (min(m, n) > 128 crossover)
        a = rng.standard_normal((n, n)) @ np.diag(np.exp(-np.arange(n) / 20)) @ rng.standard_normal((n, n))
        assert np.array_equal(cpqr_pivots_restated(a), oracle_column_pivoted_qr(a)[2])


def test_exact_ties_pick_the_first_column():
    """linalg.py:9-10: exact column-norm ties resolve to the lowest index."""
    m = make_input(CPQR_CASES["cpqr_ties_9x6"])
    norms = (m * m).sum(axis=0)
    assert np.all(norms == norms[0])
    assert cpqr_pivots_restated(m)[0] == 0 == oracle_column_pivoted_qr(m)[2][0]


def test_oracle_cor_utv_is_the_reference(reference_pkg):
    rng = np.random.default_rng(1)
    a = rng.standard_normal((120, 90)) @ np.diag(np.exp(-np.arange(90) / 10)) @ rng.standard_normal((90, 90))
    for pe in (False, True):
        for reorth in (True, False):
            ref = reference_pkg.cor_utv(a, 15, q=1, seed=4, pass_efficient=pe, reorthonormalize=reorth)
            o = oracle_cor_utv(a, 15, q=1, seed=4, pass_efficient=pe, reorthonormalize=reorth)
            assert np.array_equal(ref.u, o["u"]) and np.array_equal(ref.t, o["t"]) and np.array_equal(ref.v, o["v"])
            assert ref.sketch.passes_over_a == o["passes"] and ref.pinv_truncated == o["pinv_truncated"]
