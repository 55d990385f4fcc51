"""GPU PbP-QLP against the reference's own outputs (tests/golden/, produced by
running /root/reference's pbpqlp): same sketch, same factors within the
conditioning-aware tolerance of SURVEY.md §8 a9, same warnings and pass count."""
import json
import os
import warnings

import numpy as np
import pytest

from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, reconstruction_error
from tests.golden.recipes import CASES, make_input

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_matches_reference_fixture(cuda, name):
    from paper_2103_07245_b200 import RankDeficiencyWarning, pbp_qlp

    case = MANIFEST["cases"][name]
    a = make_input(case["recipe"])
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        f = pbp_qlp(a, case["d"], q=case["q"], seed=case["seed"], reorthonormalize=case["reorth"])
    assert sum(1 for w in rec if issubclass(w.category, RankDeficiencyWarning)) == case["rank_warnings"]
    assert f.sketch.passes_over_a == case["passes_over_a"]
    phi = f.sketch.test_matrix
    assert np.array_equal(phi, g["phi"])  # the reference's own sketch, bit for bit
    assert f.q_basis.shape == g["q"].shape and f.p_basis.shape == g["p"].shape
    assert np.array_equal(f.l, np.tril(f.l)) and np.all(np.diag(f.l) >= 0)
    assert np.array_equal(f.first_stage_r, np.triu(f.first_stage_r)) and np.all(np.diag(f.first_stage_r) >= 0)
    if case["rank_warnings"]:
        # numerically rank deficient: the reference itself warns that the
        # trailing directions are arbitrary, so compare the determined leading
        # columns (conditioning-aware tolerance ≤ 1e-6) and the warning count
        tol = conditioning_tolerance(g["l"], strict=1e-10)
        det = np.flatnonzero(np.cumprod(tol <= 1e-6))
        assert det.size >= 3
        assert np.all(column_relative_error(f.q_basis[:, det], g["q"][:, det]) <= tol[det])
        assert np.all(column_relative_error(f.p_basis[:, det], g["p"][:, det]) <= tol[det])
        lref = np.abs(np.diag(g["l"]))[det]
        ltol = conditioning_tolerance(g["l"], strict=1e-10, factor=16.0)[det]
        assert np.all(np.abs(np.diag(f.l)[det] - lref) / lref <= ltol)
        e_got = reconstruction_error(a, f.q_basis, f.l, f.p_basis)
        e_ref = reconstruction_error(a, g["q"], g["l"], g["p"])
        # both errors sit at the rounding floor (≈1e-15 of ‖A‖) here
        assert abs(e_got - e_ref) <= 1e-10 * e_ref + 1e-13
        return
    tol = conditioning_tolerance(g["l"], strict=1e-10)
    assert np.all(column_relative_error(f.q_basis, g["q"]) <= tol)
    assert np.all(column_relative_error(f.p_basis, g["p"]) <= tol)
    lref = np.abs(np.diag(g["l"]))
    assert np.all(np.abs(np.diag(f.l) - lref) / lref <= conditioning_tolerance(g["l"], strict=1e-10, factor=16.0))
    e_got = reconstruction_error(a, f.q_basis, f.l, f.p_basis)
    e_ref = reconstruction_error(a, g["q"], g["l"], g["p"])
    assert abs(e_got - e_ref) <= 1e-10 * e_ref + 1e-15


def test_nonfinite_after_valid_params(cuda):
    from paper_2103_07245_b200 import MatrixInputError, pbp_qlp

    for a in (np.full((4, 4), np.inf), np.where(np.eye(6, 5) > 0, np.nan, 1.0)):
        with pytest.raises(MatrixInputError):
            pbp_qlp(a, 2)
