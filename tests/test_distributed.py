"""Row-sharded PbP-QLP orchestration over world size 2 with
the `gloo` backend on CPU: local ops from tests/dist_backend.py, collectives
(allreduce of AᵀX, all-gather of TSQR R factors) real.  The assembled factors
must match the single-process oracle within the §8 a9 tolerance."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, a, d, q, seed, reorth, outdir, chunks=None, dist_qr="auto"):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2103_07245_b200.distributed import DistributedPbpQlp, shard_rows
    from tests.dist_backend import NumpyBackend

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, n2 = a.shape
        rows = shard_rows(n1, world)
        run = DistributedPbpQlp(n1, n2, d, q, rows, reorthonormalize=reorth, backend=NumpyBackend(), chunks=chunks,
                                dist_qr=dist_qr)
        a_loc = torch.from_numpy(np.ascontiguousarray(a[rows[rank]:rows[rank + 1]]))
        run.run(a_loc, seed=seed)
        import warnings

        with warnings.catch_warnings(record=True) as rec:
            warnings.simplefilter("always")
            run.finish()
        qg, l, p, r = run.factors()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), q=qg.numpy(), l=l.numpy(), p=p.numpy(), r=r.numpy(),
                 phi=run.PHI.numpy(), warn=len(rec), tsqr=run.tsqr_fallbacks, orthfb=run.orth_fallbacks)
    finally:
        dist.destroy_process_group()


def _run(a, d, q, seed, reorth, tmp_path, world=2, chunks=None, dist_qr="auto"):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, a, d, q, seed, reorth, str(tmp_path), chunks, dist_qr), nprocs=world,
             join=True)
    parts = [np.load(os.path.join(tmp_path, f"rank{g}.npz")) for g in range(world)]
    return parts


@pytest.mark.parametrize("q,reorth,chunks,dist_qr", [(0, True, None, "auto"), (1, True, None, "auto"),
                                                     (1, False, None, "auto"), (1, True, 3, "auto"),
                                                     (1, True, None, "tsqr")])
def test_row_sharded_matches_oracle(tmp_path, q, reorth, chunks, dist_qr):
    """chunks=3 splits AᵀX into row blocks of 128 (n2 = 300 → 128, 128, 44)
    whose allreduces are issued asynchronously while later blocks compute."""
    from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp

    rng = np.random.default_rng(11)
    n2 = 300 if chunks else 90
    a = rng.standard_normal((240, 40)) @ rng.standard_normal((40, n2)) / 7 + 1e-3 * rng.standard_normal((240, n2))
    d = 24
    parts = _run(a, d, q, 5, reorth, tmp_path, chunks=chunks, dist_qr=dist_qr)
    assert all(int(p["tsqr"]) == 0 for p in parts)  # well-conditioned: Cholesky-QR2 (or TSQR when asked)
    ref = oracle_pbp_qlp(a, d, q=q, seed=5, reorthonormalize=reorth)
    qfull = np.vstack([p["q"] for p in parts])
    phi = np.vstack([p["phi"] for p in parts])
    assert np.array_equal(phi, ref["phi"])  # sharded sketch = the global stream
    for p in parts[1:]:  # replicated factors are bitwise identical across ranks
        for k in ("l", "p", "r"):
            assert np.array_equal(p[k], parts[0][k])
    tol = conditioning_tolerance(ref["l"], strict=1e-10)
    assert np.all(column_relative_error(qfull, ref["q"]) <= tol)
    assert np.all(column_relative_error(parts[0]["p"], ref["p"]) <= tol)
    lref = np.abs(np.diag(ref["l"]))
    assert np.all(np.abs(np.diag(parts[0]["l"]) - lref) / lref <= conditioning_tolerance(ref["l"], 1e-10, 16.0))
    assert np.all(np.diag(parts[0]["l"]) >= 0) and np.all(np.diag(parts[0]["r"]) >= 0)


def test_row_sharded_rank_warning(tmp_path):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((120, 3)) @ rng.standard_normal((3, 50))
    parts = _run(a, 8, 1, 2, True, tmp_path)
    assert all(int(p["warn"]) == 3 for p in parts)  # every orth site warns on every rank
    assert all(int(p["tsqr"]) == 2 for p in parts)
    assert all(int(p["orthfb"]) == 2 for p in parts)  # ... and both orth(C) calls to the replicated QR  # rank 3 < d: the Cholesky guard hands both QRs to TSQR


def _p2p_worker(rank, world, port, a, d, q, seed, fault, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import warnings

    import torch
    import torch.distributed as dist

    from paper_2103_07245_b200 import exceptions as E
    from paper_2103_07245_b200.distributed import DistributedPbpQlp, shard_rows
    from tests.dist_backend import FakeP2PBackend

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, n2 = a.shape
        rows = shard_rows(n1, world)
        be = FakeP2PBackend(None if fault == "late_timeout" else fault)
        run = DistributedPbpQlp(n1, n2, d, q, rows, backend=be, exchange="p2p")
        a_loc = torch.from_numpy(np.ascontiguousarray(a[rows[rank]:rows[rank + 1]]))
        poisoned = ""
        if fault == "late_timeout":
            be.fault = "timeout"  # the self-check passed; a later exchange times out on rank 0
            run.run(a_loc, seed=seed)
            try:
                run.finish()
            except E.DeviceError:
                try:
                    run.run(a_loc, seed=seed)
                except E.DeviceError as exc:
                    poisoned = str(exc)
        else:
            run.run(a_loc, seed=seed)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                run.finish()
        qg, l, p, r = run.factors()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), q=qg.numpy(), l=l.numpy(), p=p.numpy(),
                 exchange=run.exchange, note=run.exchange_note, poisoned=poisoned)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fault", [None, "wrong", "timeout", "late_timeout"])
def test_p2p_self_check_and_fallback(tmp_path, fault):
    """The peer-memory exchange checks itself against NCCL-equivalent
    collectives at init (DistributedPbpQlp._p2p_self_check): a working
    transport keeps "p2p"; a wrong result on ONE rank or a spin timeout makes
    EVERY rank fall back to the collective exchange, and the factorization
    still matches the oracle.  A timeout after init poisons the exchange."""
    from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp

    rng = np.random.default_rng(13)
    a = rng.standard_normal((260, 30)) @ rng.standard_normal((30, 150)) / 6 + 1e-3 * rng.standard_normal((260, 150))
    d, q, seed, world = 20, 1, 4, 2
    port = _free_port()
    mp.spawn(_p2p_worker, args=(world, port, a, d, q, seed, fault, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(os.path.join(tmp_path, f"rank{g}.npz")) for g in range(world)]
    exch = {str(p["exchange"]) for p in parts}
    if fault in (None, "late_timeout"):
        assert exch == {"p2p"} and all("passed" in str(p["note"]) for p in parts)
    else:
        assert exch == {"nccl"} and all("self-check failed" in str(p["note"]) for p in parts)
    if fault == "late_timeout":
        assert "unusable" in str(parts[0]["poisoned"])
        return
    ref = oracle_pbp_qlp(a, d, q=q, seed=seed)
    tol = conditioning_tolerance(ref["l"], strict=1e-10)
    assert np.all(column_relative_error(np.vstack([p["q"] for p in parts]), ref["q"]) <= tol)
    assert np.all(column_relative_error(parts[0]["p"], ref["p"]) <= tol)
