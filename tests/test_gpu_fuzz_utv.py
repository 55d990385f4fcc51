"""Randomized sweep of cor_utv (algorithms.py:306-363) against the oracle:
random shapes, d, q ∈ {0, 1, 2}, both pass_efficient settings, low rank plus
noise with a spread of decay rates, judged by the checks of
tests/test_gpu_utv.py (determined block per column within the conditioning
model; structure, orthonormal bases and reconstruction error everywhere).
Reorthonormalized runs only: their intermediate orth calls are the basis-only
ones (pbq_orth_basis).  PBQ_FUZZ_CASES sets the count (default 30)."""
import os
import warnings

import numpy as np
import pytest

from oracle.pbp_qlp_oracle import oracle_cor_utv
from tests.test_gpu_utv import _check_utv

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(int(os.environ.get("PBQ_FUZZ_CASES", "30"))))
def test_random_cor_utv(cuda, seed):
    from paper_2103_07245_b200.utv import cor_utv

    rng = np.random.default_rng(12000 + seed)
    n1, n2 = int(rng.integers(60, 1800)), int(rng.integers(60, 1800))
    kmin = min(n1, n2)
    d = int(rng.integers(2, min(kmin, 200) + 1))
    q = int(rng.integers(0, 3))
    pe = bool(rng.random() < 0.5)
    r = int(min(kmin, d + rng.integers(0, 30)))
    u, _ = np.linalg.qr(rng.standard_normal((n1, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n2, r)))
    a = (u * np.exp(-np.arange(r) / float(rng.choice([8.0, 30.0, 1e9])))) @ v.T + 1e-8 * rng.standard_normal((n1, n2))
    sd = int(rng.integers(0, 2**31))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        f = cor_utv(a, d, q=q, seed=sd, pass_efficient=pe)
        ref = oracle_cor_utv(a, d, q=q, seed=sd, pass_efficient=pe)
    assert f.sketch.passes_over_a == ref["passes"], (a.shape, d, q, pe)
    _check_utv(a, f, ref["u"], ref["t"], ref["v"], ref)
