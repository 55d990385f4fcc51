"""``pbp_qlp_multi_gpu``: the single-call launcher over the row-sharded driver
 — one worker process per rank, A handed over in row blocks,
Q / L / P / R / Φ collected on the host.  Only one GPU is available to the
tests, so the ranks share cuda:0 over the ``gloo`` backend (host-mediated
collectives: no rank's kernel waits on another's); the NCCL transport itself
is the one thing this does not cover."""
import warnings

import numpy as np
import pytest

from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp

pytestmark = pytest.mark.gpu


def _matrix(seed, n1=1500, n2=700):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n1, 60)) @ rng.standard_normal((60, n2)) / 8 + 1e-3 * rng.standard_normal((n1, n2))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,q,reorth", [(2, 1, True), (3, 2, True), (2, 2, False), (2, 0, True)])
def test_matches_oracle_and_single_gpu(cuda, world, q, reorth):
    from paper_2103_07245_b200 import pbp_qlp, pbp_qlp_multi_gpu

    a = _matrix(17)
    d = 48
    got = pbp_qlp_multi_gpu(a, d, q=q, seed=9, reorthonormalize=reorth, devices=[0] * world, backend="gloo")
    ref = oracle_pbp_qlp(a, d, q=q, seed=9, reorthonormalize=reorth)
    one = pbp_qlp(a, d, q=q, seed=9, reorthonormalize=reorth)
    assert np.array_equal(got.sketch.test_matrix, ref["phi"])  # the sharded device sketch: bit-exact
    assert (got.sketch.seed, got.sketch.d, got.sketch.q, got.sketch.passes_over_a) == (9, d, q, 2 * q + 2)
    tol = conditioning_tolerance(ref["l"], strict=1e-10)
    for x, o, s in ((got.q_basis, ref["q"], one.q_basis), (got.p_basis, ref["p"], one.p_basis)):
        assert np.all(column_relative_error(x, o) <= tol)
        assert np.all(column_relative_error(x, s) <= tol)
    lref = np.abs(np.diag(ref["l"]))
    assert np.all(np.abs(np.abs(np.diag(got.l)) - lref) / lref <= conditioning_tolerance(ref["l"], 1e-10, 16.0))
    recon = np.linalg.norm(a - got.q_basis @ got.l @ got.p_basis.T) / np.linalg.norm(a)
    ref_recon = np.linalg.norm(a - ref["q"] @ ref["l"] @ ref["p"].T) / np.linalg.norm(a)
    assert abs(recon - ref_recon) <= 1e-10


@pytest.mark.timeout(600)
def test_warnings_and_errors_are_the_reference_ones(cuda):
    from paper_2103_07245_b200 import MatrixInputError, ParameterError, RankDeficiencyWarning, pbp_qlp_multi_gpu

    rng = np.random.default_rng(3)
    low = rng.standard_normal((600, 3)) @ rng.standard_normal((3, 200))
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        pbp_qlp_multi_gpu(low, 8, q=1, seed=2, devices=[0, 0], backend="gloo")
    assert sum(issubclass(w.category, RankDeficiencyWarning) for w in rec) == 3  # every orth site, once
    bad = _matrix(5, 400, 300)
    bad[250, 7] = np.nan  # in rank 1's rows
    with pytest.raises(MatrixInputError):
        pbp_qlp_multi_gpu(bad, 16, q=1, devices=[0, 0], backend="gloo")
    with pytest.raises(MatrixInputError):  # A is validated before d (algorithms.py:239-241)
        pbp_qlp_multi_gpu(bad, 0, devices=[0, 0], backend="gloo")
    with pytest.raises(ParameterError):
        pbp_qlp_multi_gpu(_matrix(5, 400, 300), 301, devices=[0, 0], backend="gloo")
    with pytest.raises(ParameterError):
        pbp_qlp_multi_gpu(_matrix(5, 400, 300), 16, devices=[0, 0], backend="nccl")  # one GPU per NCCL rank


@pytest.mark.timeout(600)
def test_short_matrices_use_fewer_ranks(cuda):
    from paper_2103_07245_b200 import pbp_qlp, pbp_qlp_multi_gpu
    from paper_2103_07245_b200.multigpu import usable_world

    assert usable_world(1000, 40, 8) == 8 and usable_world(100, 40, 8) == 2 and usable_world(50, 40, 8) == 1
    a = _matrix(7, 90, 300)
    got = pbp_qlp_multi_gpu(a, 64, q=1, seed=4, devices=[0, 0, 0], backend="gloo")  # 90 // 2 < 64: one rank
    one = pbp_qlp(a, 64, q=1, seed=4)
    assert np.array_equal(got.q_basis, one.q_basis) and np.array_equal(got.l, one.l)


@pytest.mark.timeout(600)
def test_reference_callers_reach_the_launcher(cuda, reference_pkg):
    """integration.install(pbpqlp, devices=…): the reference's own entry point,
    result types and warnings, computed by the sharded ranks."""
    from paper_2103_07245_b200 import integration

    a = _matrix(23, 900, 500)
    saved = integration.install(reference_pkg, devices=[0, 0], backend="gloo")
    try:
        f = reference_pkg.pbp_qlp(a, 40, q=1, seed=5)
        pool = reference_pkg.pbp_qlp.__pool_holder__["pool"]
        f2 = reference_pkg.pbp_qlp(a, 40, q=1, seed=6)  # the same workers serve the next call
        assert reference_pkg.pbp_qlp.__pool_holder__["pool"] is pool and len(pool.procs) == 2
        assert not np.array_equal(f2.sketch.test_matrix, f.sketch.test_matrix)
    finally:
        integration.uninstall(saved)
    assert pool.procs == []  # uninstall stopped them
    assert type(f).__module__.startswith("pbpqlp")
    ref = reference_pkg.pbp_qlp(a, 40, q=1, seed=5)
    tol = conditioning_tolerance(ref.l, strict=1e-10)
    assert np.array_equal(f.sketch.test_matrix, ref.sketch.test_matrix)
    assert np.all(column_relative_error(f.q_basis, ref.q_basis) <= tol)
    assert np.all(column_relative_error(f.p_basis, ref.p_basis) <= tol)
    assert f.sketch.passes_over_a == ref.sketch.passes_over_a == 4


@pytest.mark.timeout(300)
def test_a_failing_rank_fails_the_call(cuda):
    """A rank that raises takes the job down (no rank is left waiting in a
    collective) and the parent reports what the rank recorded."""
    from paper_2103_07245_b200 import DeviceError, pbp_qlp_multi_gpu

    with pytest.raises(DeviceError, match="rank"):
        # an exchange name the sharded driver rejects: every rank raises in its constructor
        pbp_qlp_multi_gpu(_matrix(5, 400, 300), 16, q=1, devices=[0, 0], backend="gloo", exchange="bogus")


@pytest.mark.timeout(600)
def test_pool_serves_many_calls(cuda):
    """MultiGpuPool: the workers start once and serve several factorizations
    (different seeds and shapes, a NaN input in between), each equal to the
    one-shot call's contract."""
    from paper_2103_07245_b200 import MatrixInputError, MultiGpuPool, pbp_qlp

    a = _matrix(31, 1200, 600)
    b = _matrix(32, 800, 900)
    with MultiGpuPool([0, 0], backend="gloo") as pool:
        assert pool.world == 2
        for m, d, q, seed in ((a, 40, 1, 1), (a, 40, 1, 2), (b, 64, 2, 3), (a, 40, 1, 1)):
            got = pool.pbp_qlp(m, d, q=q, seed=seed)
            one = pbp_qlp(m, d, q=q, seed=seed)
            ref = oracle_pbp_qlp(m, d, q=q, seed=seed)
            tol = conditioning_tolerance(ref["l"], strict=1e-10)
            assert np.array_equal(got.sketch.test_matrix, ref["phi"])
            assert np.all(column_relative_error(got.q_basis, ref["q"]) <= tol)
            assert np.all(column_relative_error(got.p_basis, one.p_basis) <= tol)
        bad = a.copy()
        bad[1000, 3] = np.inf
        with pytest.raises(MatrixInputError):
            pool.pbp_qlp(bad, 40, q=1)
        again = pool.pbp_qlp(a, 40, q=1, seed=1)  # the pool survives a rejected input
        assert np.array_equal(again.sketch.test_matrix, oracle_pbp_qlp(a, 40, q=1, seed=1)["phi"])
        short = pool.pbp_qlp(_matrix(7, 90, 300), 64, q=1, seed=4)  # too short to shard: the single-GPU path
        assert short.q_basis.shape == (90, 64)
    assert pool.procs == []
