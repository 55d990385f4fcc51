"""Pins the CPU oracle (oracle/) before it is trusted as the parity checker:
against the reference's golden fixtures (tests/golden/, made by running
/root/reference's pbpqlp), against the reference itself when it is importable,
and the C sketch restatement against numpy's Generator bit for bit."""
import json
import os

import numpy as np
import pytest

from oracle.pbp_qlp_oracle import (
    c_gaussian,
    c_philox_raw,
    column_relative_error,
    conditioning_tolerance,
    householder_qr_restated,
    oracle_gaussian,
    oracle_pbp_qlp,
    oracle_qr,
)
from tests.golden.recipes import CASES, make_input

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


def _sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_golden(name):
    case = MANIFEST["cases"][name]
    a = make_input(case["recipe"])
    assert _sha(a) == case["a_sha256"], "input recipe no longer reproduces the fixture's A"
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    o = oracle_pbp_qlp(a, case["d"], q=case["q"], seed=case["seed"], reorthonormalize=case["reorth"])
    assert np.array_equal(o["phi"], g["phi"])  # the sketch is bit-exact everywhere
    assert o["passes"] == case["passes_over_a"]
    assert sum(1 for f in o["rank_flags"] if f) == case["rank_warnings"]
    if case["rank_warnings"]:
        return  # trailing directions are arbitrary by construction
    tol = conditioning_tolerance(g["l"], strict=1e-11)
    assert np.all(column_relative_error(o["q"], g["q"]) <= tol)
    assert np.all(column_relative_error(o["p"], g["p"]) <= tol)
    assert np.allclose(np.abs(np.diag(o["l"])), np.abs(np.diag(g["l"])), rtol=1e-11, atol=0)


def test_oracle_is_the_reference(reference_pkg):
    """Call-for-call restatement: bitwise equal to pbpqlp on the same machine."""
    rng = np.random.default_rng(0)
    a = rng.standard_normal((300, 200))
    for q in (0, 2):
        for reorth in (True, False):
            ref = reference_pkg.pbp_qlp(a, 25, q=q, seed=3, reorthonormalize=reorth)
            o = oracle_pbp_qlp(a, 25, q=q, seed=3, reorthonormalize=reorth)
            for x, y in ((ref.q_basis, o["q"]), (ref.l, o["l"]), (ref.p_basis, o["p"]), (ref.first_stage_r, o["r"]),
                         (ref.sketch.test_matrix, o["phi"])):
                assert np.array_equal(x, y)
            assert ref.sketch.passes_over_a == o["passes"]


@pytest.mark.parametrize("key", sorted(MANIFEST["sketches"]))
def test_sketch_golden(key):
    meta = MANIFEST["sketches"][key]
    g = np.load(os.path.join(GOLDEN, key + ".npy"))
    assert np.array_equal(oracle_gaussian(meta["rows"], meta["cols"], meta["seed"]), g)
    assert np.array_equal(c_gaussian(meta["rows"], meta["cols"], meta["seed"]), g)


@pytest.mark.parametrize("seed", [0, 1, 42, 2**64 + 3, 2**127 + 99])
def test_c_sketch_matches_numpy(seed):
    raw = np.random.Philox(key=seed).random_raw(4096)
    assert np.array_equal(c_philox_raw(seed, 0, 4096), raw)
    n = 200_000
    ref = np.random.Generator(np.random.Philox(key=seed)).standard_normal(n)
    out = c_gaussian(1, n, seed)[0]
    assert np.array_equal(out, ref)


def test_c_sketch_row_offset():
    full = oracle_gaussian(500, 37, 11)
    assert np.array_equal(c_gaussian(123, 37, 11, row_offset=250), full[250:373])


@pytest.mark.parametrize("shape", [(50, 10), (200, 64), (33, 33), (100, 1)])
def test_restated_householder_matches_lapack(shape):
    a = np.random.default_rng(shape[0]).standard_normal(shape)
    q1, r1 = oracle_qr(a)
    q2, r2 = householder_qr_restated(a)
    assert np.abs(q1 - q2).max() < 1e-13
    assert np.abs(r1 - r2).max() < 1e-12 * np.abs(r1).max()


def test_log1p_restatement_is_the_c_library():
    """The sketch's exponential tail calls log1p (numpy's npy_log1p → the C
    library).  The device restates glibc's (sketch.cuh: glibc_log1p); its
    host twin must equal libm bit for bit on the sampler's domain
    x = −k·2⁻⁵³ ∈ (−1, 0] and across every branch of the function."""
    from oracle.pbp_qlp_oracle import c_log1p_pair

    rng = np.random.default_rng(2024)
    dom = -(rng.integers(0, 2**53, size=2_000_000, dtype=np.int64).astype(np.float64) * 2.0**-53)
    e = np.arange(-70, 0)
    m = np.linspace(1.0, 2.0, 400, endpoint=False)
    edges = (m[None, :] * np.ldexp(1.0, e)[:, None]).ravel()
    wide = np.concatenate([rng.uniform(-1, 8, 200_000), np.ldexp(rng.uniform(1, 2, 20_000), rng.integers(-60, 60, 20_000))])
    x = np.concatenate([dom, -edges[edges < 1], edges, wide, [0.0, -0.0, 0.41422, -0.2929, 1e300, -1.0 + 2**-53]])
    mine, libm = c_log1p_pair(x)
    bad = np.flatnonzero(mine.view(np.int64) != libm.view(np.int64))
    assert bad.size == 0, (x[bad[:5]], mine[bad[:5]], libm[bad[:5]])
