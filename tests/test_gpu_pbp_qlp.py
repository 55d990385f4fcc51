"""End-to-end parity of the GPU PbP-QLP against the CPU oracle (which is the
reference's numpy call sequence, algorithms.py:209-260) and the reference
test suite's properties (tests/test_algorithms.py of the reference)."""
import warnings

import numpy as np
import pytest
import torch

from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp, reconstruction_error

pytestmark = pytest.mark.gpu


def _check_against_oracle(a, d, q, seed, reorth=True, phi=None, strict=1e-10, ncols=None):
    """``ncols`` limits the column checks to the numerically determined
    leading directions (when the oracle itself warns that the trailing basis
    directions are arbitrary)."""
    from paper_2103_07245_b200 import pbp_qlp

    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        got = pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorth, phi=phi)
    ref = oracle_pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorth, phi=phi)
    assert sum(1 for w in rec if "orth:" in str(w.message)) == sum(1 for f in ref["rank_flags"] if f)
    k = d if ncols is None else ncols
    tol = conditioning_tolerance(ref["l"], strict=strict)[:k]
    assert np.all(column_relative_error(got.q_basis[:, :k], ref["q"][:, :k]) <= tol)
    assert np.all(column_relative_error(got.p_basis[:, :k], ref["p"][:, :k]) <= tol)
    lref = np.abs(np.diag(ref["l"]))[:k]
    lerr = np.abs(np.abs(np.diag(got.l))[:k] - lref) / np.where(lref > 0, lref, 1.0)
    assert np.all(lerr <= conditioning_tolerance(ref["l"], strict=strict, factor=16.0)[:k])
    e_got = reconstruction_error(a, got.q_basis, got.l, got.p_basis)
    e_ref = reconstruction_error(a, ref["q"], ref["l"], ref["p"])
    if ncols is None:  # with arbitrary trailing directions the error itself is arbitrary at O(σ_noise)
        assert abs(e_got - e_ref) <= 1e-10 * max(e_ref, 1e-300) + 1e-15
    assert got.sketch.passes_over_a == ref["passes"] == 2 * q + 2
    return got, ref


def test_small_seeded(cuda):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((300, 200))
    got, ref = _check_against_oracle(a, 25, 1, 3)
    assert np.array_equal(got.sketch.test_matrix, ref["phi"])


@pytest.mark.parametrize("q,reorth", [(0, True), (2, True), (0, False), (2, False)])
def test_low_rank_plus_noise(cuda, qr_method, q, reorth):
    rng = np.random.default_rng(7)
    a = rng.standard_normal((800, 30)) @ rng.standard_normal((30, 500)) / 30 + 1e-4 * rng.standard_normal((800, 500))
    # without re-orthonormalization the q=2 sketch squares the spectrum twice:
    # the 10 noise directions fall below eps and are arbitrary in both codes
    _check_against_oracle(a, 40, q, 5, reorth=reorth, ncols=30 if (q and not reorth) else None)


def test_structure(cuda):
    from paper_2103_07245_b200 import pbp_qlp

    rng = np.random.default_rng(1)
    a = rng.standard_normal((120, 90))
    f = pbp_qlp(a, 20, q=1, seed=2)
    assert f.q_basis.shape == (120, 20) and f.l.shape == (20, 20)
    assert f.p_basis.shape == (90, 20) and f.first_stage_r.shape == (20, 20)
    assert np.abs(f.q_basis.T @ f.q_basis - np.eye(20)).max() < 1e-11
    assert np.abs(f.p_basis.T @ f.p_basis - np.eye(20)).max() < 1e-11
    assert np.array_equal(f.l, np.tril(f.l))
    assert np.array_equal(f.first_stage_r, np.triu(f.first_stage_r))
    assert np.all(np.diag(f.l) >= 0)


def test_determinism_and_seed(cuda):
    from paper_2103_07245_b200 import pbp_qlp

    rng = np.random.default_rng(2)
    a = rng.standard_normal((500, 300))
    f1 = pbp_qlp(a, 30, q=1, seed=4)
    f2 = pbp_qlp(a, 30, q=1, seed=4)
    f3 = pbp_qlp(a, 30, q=1, seed=5)
    assert np.array_equal(f1.l, f2.l) and np.array_equal(f1.q_basis, f2.q_basis)
    assert not np.array_equal(f1.l, f3.l)


def test_rank_deficiency_warning(cuda):
    from paper_2103_07245_b200 import RankDeficiencyWarning, pbp_qlp

    rng = np.random.default_rng(3)
    a = rng.standard_normal((200, 4)) @ rng.standard_normal((4, 150))
    with pytest.warns(RankDeficiencyWarning):
        pbp_qlp(a, 10)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        pbp_qlp(rng.standard_normal((200, 150)), 10)


def test_nonfinite_raises(cuda):
    from paper_2103_07245_b200 import MatrixInputError, pbp_qlp

    a = np.ones((64, 48))
    a[63, 47] = np.nan
    with pytest.raises(MatrixInputError):
        pbp_qlp(a, 4)


def test_torch_input_stays_on_device(cuda):
    from paper_2103_07245_b200 import pbp_qlp

    a = torch.randn(400, 300, dtype=torch.float64, device=cuda)
    f = pbp_qlp(a, 32, q=1)
    assert isinstance(f.q_basis, torch.Tensor) and f.q_basis.is_cuda
    ref = pbp_qlp(a.cpu().numpy(), 32, q=1)
    assert np.array_equal(f.l.cpu().numpy(), ref.l)


def test_integration_shim_returns_reference_types(cuda):
    """The drop-in wrapper hands back the reference's dataclasses; a stand-in
    module with the reference's attribute layout replaces the reference here
    (it is not present on the GPU box)."""
    import types
    from dataclasses import dataclass
    from typing import Any

    from paper_2103_07245_b200 import integration

    @dataclass(frozen=True)
    class SketchRecord:
        test_matrix: Any
        seed: int
        d: int
        q: int
        passes_over_a: int

    @dataclass(frozen=True)
    class QlpFactors:
        q_basis: Any
        l: Any
        p_basis: Any
        first_stage_r: Any
        sketch: Any = None

    @dataclass(frozen=True)
    class RsvdFactors:
        u: Any
        s: Any
        v: Any
        sketch: Any

    class ParameterError(ValueError):
        pass

    class DimensionError(ParameterError):
        pass

    class MatrixInputError(ValueError):
        pass

    class RankDeficiencyWarning(UserWarning):
        pass

    fake = types.SimpleNamespace(
        algorithms=types.SimpleNamespace(SketchRecord=SketchRecord, QlpFactors=QlpFactors, RsvdFactors=RsvdFactors,
                                         pbp_qlp=lambda *a, **k: None, r_svd=lambda *a, **k: None),
        exceptions=types.SimpleNamespace(ParameterError=ParameterError, DimensionError=DimensionError,
                                         MatrixInputError=MatrixInputError, RankDeficiencyWarning=RankDeficiencyWarning),
    )
    fn = integration.make_dropin(fake)
    rng = np.random.default_rng(4)
    a = rng.standard_normal((200, 120))
    f = fn(a, 16, q=1, seed=3)
    assert isinstance(f, QlpFactors) and isinstance(f.sketch, SketchRecord)
    assert f.sketch.passes_over_a == 4 and f.sketch.test_matrix.shape == (200, 16)
    with pytest.raises(ParameterError):
        fn(a, 500)
    rs = integration.make_rsvd_dropin(fake)
    g = rs(a, 16, q=1, seed=3)
    assert isinstance(g, RsvdFactors) and isinstance(g.sketch, SketchRecord)
    assert g.sketch.passes_over_a == 4 and g.sketch.test_matrix.shape == (120, 16) and g.u.shape == (200, 16)
    with pytest.raises(ParameterError):
        rs(a, 500)
    low = rng.standard_normal((200, 3)) @ rng.standard_normal((3, 120))
    with pytest.warns(RankDeficiencyWarning):
        fn(low, 10)


def test_distributed_driver_on_one_gpu(cuda):
    """The row-sharded driver with NCCL and the CUDA backend (world size 1 on
    the single-GPU box): TSQR + allreduce path against the fused pipeline."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2103_07245_b200 import pbp_qlp
    from paper_2103_07245_b200.distributed import DistributedPbpQlp, shard_rows

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=cuda)
    try:
        rng = np.random.default_rng(9)
        a = rng.standard_normal((900, 60)) @ rng.standard_normal((60, 500)) / 8 + 1e-3 * rng.standard_normal((900, 500))
        at = torch.from_numpy(a).to(cuda)
        ref = pbp_qlp(a, 48, q=1, seed=7)
        tol = conditioning_tolerance(ref.l, strict=1e-10)
        for chunks in (1, 3):  # 3: AᵀX in 128-row blocks with asynchronous NCCL allreduces
            run = DistributedPbpQlp(900, 500, 48, 1, shard_rows(900, 1), device=cuda, chunks=chunks)
            run.run(at, seed=7)
            run.finish()
            qg, l, p, r = (t.cpu().numpy() for t in run.factors())
            assert np.all(column_relative_error(qg, ref.q_basis) <= tol)
            assert np.all(column_relative_error(p, ref.p_basis) <= tol)
            assert np.allclose(np.diag(l), np.diag(ref.l), rtol=1e-10, atol=0)
            # the same step captured as a CUDA graph (kernels + NCCL
            # collectives) and replayed: bitwise the stream-ordered result
            run.capture(at, seed=7)
            for t in run.factors():
                t.fill_(float("nan"))
            run.replay()
            run.finish()
            for x, y in zip((t.cpu().numpy() for t in run.factors()), (qg, l, p, r)):
                assert np.array_equal(x, y)
            assert run.graph_launches > 0
    finally:
        dist.destroy_process_group()


def test_streamed_host_path_matches_oracle(cuda, monkeypatch):
    """Host inputs above STREAM_MIN_BYTES stream to the device in row chunks
    overlapped with the first pass; force it on a small case (pinned torch
    and numpy inputs) and check parity with the oracle."""
    from paper_2103_07245_b200 import algorithms

    monkeypatch.setattr(algorithms, "STREAM_MIN_BYTES", 0)
    rng = np.random.default_rng(12)
    a = rng.standard_normal((1500, 50)) @ rng.standard_normal((50, 700)) / 7 + 1e-3 * rng.standard_normal((1500, 700))
    got_np, ref = _check_against_oracle(a, 40, 1, 21)
    assert isinstance(got_np.q_basis, np.ndarray)
    ta = torch.from_numpy(a).pin_memory()
    got_t = algorithms.pbp_qlp(ta, 40, q=1, seed=21)
    assert isinstance(got_t.q_basis, torch.Tensor) and not got_t.q_basis.is_cuda
    assert np.array_equal(got_t.l.numpy(), got_np.l)
    bad = a.copy()
    bad[1499, 3] = np.inf
    from paper_2103_07245_b200 import MatrixInputError

    with pytest.raises(MatrixInputError):
        algorithms.pbp_qlp(bad, 40, q=1)
