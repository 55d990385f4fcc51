"""Parity at BASELINE.json sizes and edge shapes:
configs 2 and 3 at full size, config-5 analogs up to d = 1024, d = min(n1, n2),
wide A, many power iterations.  Tolerance per column: max(1e-10, 64·u·κ_j)
for Q and P, max(1e-10, 16·u·κ_j) for |diag L| (κ_j = L_00/L_jj), and the
relative reconstruction error within 1e-10."""
import math
import warnings

import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp

pytestmark = pytest.mark.gpu


def _recon_err(a_dev, qf, l, p):
    """‖A − QLPᵀ‖_F / ‖A‖_F in FP64 on the device (torch, test-side check)."""
    qf, l, p = (torch.as_tensor(x, device=a_dev.device) for x in (qf, l, p))
    return float(torch.linalg.norm(a_dev - qf @ l @ p.T) / torch.linalg.norm(a_dev))


def _parity(a_host, d, q, seed, a_dev=None, strict=1e-10):
    from paper_2103_07245_b200 import pbp_qlp

    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        got = pbp_qlp(a_dev if a_dev is not None else a_host, d, q=q, seed=seed)
    ref = oracle_pbp_qlp(a_host, d, q=q, seed=seed)
    assert sum(1 for w in rec if "orth:" in str(w.message)) == sum(1 for f in ref["rank_flags"] if f)
    gq, gl, gp = (x.cpu().numpy() if isinstance(x, torch.Tensor) else x for x in (got.q_basis, got.l, got.p_basis))
    tol = conditioning_tolerance(ref["l"], strict=strict)
    eq = column_relative_error(gq, ref["q"])
    ep = column_relative_error(gp, ref["p"])
    assert np.all(eq <= tol), (eq.max(), np.argmax(eq / tol))
    assert np.all(ep <= tol), (ep.max(), np.argmax(ep / tol))
    lref = np.abs(np.diag(ref["l"]))
    el = np.abs(np.diag(gl) - lref) / lref
    assert np.all(el <= conditioning_tolerance(ref["l"], strict=strict, factor=16.0))
    ad = a_dev if a_dev is not None else torch.from_numpy(a_host).cuda()
    e_got = _recon_err(ad, gq, gl, gp)
    e_ref = _recon_err(ad, ref["q"], ref["l"], ref["p"])
    assert abs(e_got - e_ref) <= 1e-10 * e_ref + 1e-15
    # the fused one-pass residual agrees with the dense check
    from paper_2103_07245_b200 import reconstruction_error

    assert abs(reconstruction_error(ad, got) - e_got) <= 1e-10 * e_got + 1e-15
    return eq.max(), ep.max()


def test_config2_full(cuda):
    from paper_2103_07245_b200 import workloads

    a = workloads.make_cfg2(0)
    _parity(a, 100, 0, 0)


def test_config3_full(cuda):
    from paper_2103_07245_b200 import workloads

    a_dev = workloads.make_cfg3(0, cuda)
    a = a_dev.cpu().numpy()
    _parity(a, 256, 1, 0, a_dev=a_dev)


@pytest.mark.parametrize("d,q", [(64, 0), (256, 2), (512, 0), (1024, 2)])
def test_config5_analog(cuda, d, q):
    """16384×4096 with config 5's spectrum law (σ_i = e^(−i/40) over inner
    dimension 2048, + 1e-8·N(0,1)): the conditioning-limited case."""
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    n1, n2, k = 16384, 4096, 2048
    gu = torch.randn(n1, k, dtype=torch.float64, device=cuda, generator=g)
    gv = torch.randn(n2, k, dtype=torch.float64, device=cuda, generator=g)
    sigma = torch.exp(-torch.arange(k, dtype=torch.float64, device=cuda) / 40.0)
    a_dev = torch.randn(n1, n2, dtype=torch.float64, device=cuda, generator=g).mul_(1e-8)
    a_dev.addmm_(gu * sigma, gv.T, alpha=1.0 / math.sqrt(n1))
    _parity(a_dev.cpu().numpy(), d, q, 3, a_dev=a_dev)


def test_full_rank_d_equals_min_dim(cuda):
    rng = np.random.default_rng(21)
    a = rng.standard_normal((300, 200))
    _parity(a, 200, 1, 4)


def test_wide_matrix(cuda):
    rng = np.random.default_rng(22)
    a = rng.standard_normal((150, 700))
    _parity(a, 100, 1, 6)


def test_many_power_iterations(cuda):
    rng = np.random.default_rng(23)
    a = rng.standard_normal((700, 40)) @ rng.standard_normal((40, 500)) + 1e-2 * rng.standard_normal((700, 500))
    _parity(a, 48, 5, 8)


def test_odd_everything(cuda):
    rng = np.random.default_rng(24)
    a = rng.standard_normal((333, 257))
    _parity(a, 65, 1, 2**90 + 17)


@pytest.mark.slow
def test_config4_full(cuda):
    """Config 4 at its BASELINE size: 200000×8192 (A = 13.1 GB), d = 512, q = 1,
    σ_i = 10^(−i/128).  The oracle runs on the box's host cores (~1 min)."""
    from paper_2103_07245_b200 import workloads

    a_dev = workloads.make_cfg4(0, cuda)
    a = a_dev.cpu().numpy()
    _parity(a, 512, 1, 0, a_dev=a_dev)


@pytest.fixture(scope="module")
def cfg5_matrix(cuda):
    """Config 5's A (65536×16384, 8.6 GB) on the device and its host copy,
    built once for the whole d-sweep."""
    from paper_2103_07245_b200 import workloads

    a_dev = workloads.make_cfg5(0, cuda)
    a = a_dev.cpu().numpy()
    yield a_dev, a
    del a_dev
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("q", [0, 2])
@pytest.mark.parametrize("d", [64, 128, 256, 512, 1024])
def test_config5_full(cuda, cfg5_matrix, d, q):
    """Config 5 at its BASELINE size, every point of the d-sweep the bench
    reports (BASELINE.json configs[4]): 65536×16384 (A = 8.6 GB),
    σ_i = e^(−i/40) over inner dimension 2048 + 1e-8·N(0,1),
    d ∈ {64, 128, 256, 512, 1024}, q ∈ {0, 2}.  d ≥ 512 is conditioning-
    limited: the per-column bound is max(1e-10, 64·u·κ_j)."""
    a_dev, a = cfg5_matrix
    _parity(a, d, q, 0, a_dev=a_dev)
