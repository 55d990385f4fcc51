"""The fused AᵀX exchange over peer memory (distributed.py / exchange_f64.cuh:
scatter-epilogue GEMM → slice reduce + all-gather → wait), the p2p
alternative to GEMM + ncclAllReduce.

One GPU is available, so two checks:
* virtual ranks: G buffer sets on one device whose "peer" pointers refer to
  each other (distributed.virtual_exchanges).  Every virtual rank's scatter
  GEMM runs first, then every reduce, then every wait, so no kernel ever
  spins on a kernel that has not run: the data movement, slot indexing,
  slice ownership, fixed-order sums and the monotonic counter targets are
  exercised on the real kernels for G = 1…4, over two epochs;
* a real world-1 process group: the driver with exchange="p2p" allocates its
  buffers in torch symmetric memory and factors A, checked against the
  oracle like the NCCL path.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("n2,d", [(1000, 100), (700, 256), (333, 40)])
def test_virtual_rank_exchange(cuda, world, n2, d):
    from paper_2103_07245_b200 import device as D
    from paper_2103_07245_b200.distributed import shard_rows, virtual_exchanges

    ctx = D.context(cuda)
    rng = np.random.default_rng(world * 100 + d)
    n1 = 900
    xs = virtual_exchanges(n2, d, world, cuda)
    rows = shard_rows(n1, world)
    for epoch in (1, 2):
        a = rng.standard_normal((n1, n2))
        x = rng.standard_normal((n1, d))
        if epoch == 2:
            a[rows[-2] + 1, 3] = np.inf  # a non-finite entry in the last shard
        flags = torch.zeros(world, dtype=torch.int32, device=cuda)
        for g in range(world):
            ag = D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(a[rows[g]:rows[g + 1]])).to(cuda))
            xg = D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(x[rows[g]:rows[g + 1]])).to(cuda))
            D.gemm_tn_scatter(ctx, ag, xg, xs[g], nonfinite=flags[g:g + 1])
        for r in range(world):
            tiles = D.xchg_expected_tiles(ctx, n2, d, xs[r].S, r, world)
            D.xchg_reduce(ctx, xs[r], n2, d, epoch * tiles)
        for r in range(world):
            D.xchg_wait(ctx, xs[r], epoch * 64 * world)
        torch.cuda.synchronize()
        got = [xs[r].C[:n2, :d].cpu().numpy() for r in range(world)]
        for r in range(1, world):
            assert np.array_equal(got[r], got[0], equal_nan=True)  # one owner per slice: identical everywhere
        if epoch == 2:
            assert flags.cpu().tolist()[world - 1] == 1
            continue
        assert flags.cpu().tolist() == [0] * world
        ref = a.T @ x
        bound = 4 * n1 * 2.0**-53 * (np.abs(a.T) @ np.abs(x))
        assert np.all(np.abs(got[0] - ref) <= bound)
        assert int(xs[0].cnt.item()) == epoch * D.xchg_expected_tiles(ctx, n2, d, xs[0].S, 0, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, a, d, q, seed, outdir, reps=2):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2103_07245_b200 import device as D
    from paper_2103_07245_b200.distributed import DistributedPbpQlp, shard_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        n1, n2 = a.shape
        rows = shard_rows(n1, world)
        run = DistributedPbpQlp(n1, n2, d, q, rows, device=dev, exchange="p2p")
        a_loc = D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(a[rows[rank]:rows[rank + 1]])).to(dev))
        import warnings

        for _ in range(reps):  # repeated factorizations: later epochs of the exchange
            with warnings.catch_warnings(record=True) as rec:
                warnings.simplefilter("always")
                run.run(a_loc, seed=seed)
                run.finish()
        qg, l, p, r = (t.cpu().numpy() for t in run.factors())
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), q=qg, l=l, p=p, epoch=run.epoch, tsqr=run.tsqr_fallbacks,
                 warn=len(rec), exchange=run.exchange, note=run.exchange_note)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_p2p_driver_world1_matches_oracle(cuda, tmp_path):
    from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp

    rng = np.random.default_rng(23)
    n1, n2, d, q = 1500, 700, 48, 1
    a = rng.standard_normal((n1, 60)) @ rng.standard_normal((60, n2)) / 8 + 1e-3 * rng.standard_normal((n1, n2))
    mp.spawn(_worker, args=(1, _free_port(), a, d, q, 9, str(tmp_path)), nprocs=1, join=True)
    part = np.load(os.path.join(tmp_path, "rank0.npz"))
    # the init self-check (one AᵀX exchange vs an NCCL allreduce) passed on the
    # real symmetric-memory buffers; then q+1 exchanges per factorization, two factorizations
    assert str(part["exchange"]) == "p2p" and "passed" in str(part["note"]), str(part["note"])
    assert int(part["epoch"]) == 1 + 2 * (q + 1)
    ref = oracle_pbp_qlp(a, d, q=q, seed=9)
    tol = conditioning_tolerance(ref["l"], strict=1e-10)
    assert np.all(column_relative_error(part["q"], ref["q"]) <= tol)
    assert np.all(column_relative_error(part["p"], ref["p"]) <= tol)


@pytest.mark.timeout(120)
def test_exchange_wait_times_out_instead_of_hanging(cuda):
    """A peer that never arrives: the wait gives up after 20 s and reports it."""
    import time

    from paper_2103_07245_b200 import device as D
    from paper_2103_07245_b200.distributed import virtual_exchanges

    ctx = D.context(cuda)
    (x,) = virtual_exchanges(256, 16, 1, cuda)
    t0 = time.time()
    D.xchg_wait(ctx, x, 1 << 30)
    torch.cuda.synchronize()
    assert 15 < time.time() - t0 < 60
    assert int(x.status.item()) == 1


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_virtual_rank_small_collectives(cuda, world):
    """The Gram allreduce (push into every rank's slot, slot-ordered sum; two
    epochs, i.e. both halves of the double-buffered slots) and the all-gather
    of the C row slices, on virtual ranks in emulation order."""
    from paper_2103_07245_b200.distributed import CudaBackend, virtual_exchanges

    be = CudaBackend(cuda)
    n2, d = 1000, 100
    xs = virtual_exchanges(n2, d, world, cuda)
    npad = 128  # the Gram's padded size for d = 100
    rng = np.random.default_rng(world)
    for epoch in (1, 2, 3):
        gs = [torch.from_numpy(rng.standard_normal((npad, npad))).to(cuda) for _ in range(world)]
        ref = sum(g.cpu().numpy() for g in gs)
        for r in range(world):
            be.p2p_allreduce_push(xs[r], gs[r], epoch)
        for r in range(world):
            be.p2p_allreduce_sum(xs[r], gs[r], epoch)
        torch.cuda.synchronize()
        out = [g.cpu().numpy() for g in gs]
        for r in range(world):
            assert np.array_equal(out[r], out[0])
        assert np.abs(out[0] - ref).max() <= 1e-12 * np.abs(ref).max()
    for epoch in (1, 2):
        slices = []
        for r in range(world):
            sl = torch.from_numpy(rng.standard_normal((xs[r].S, xs[r].ldl))).to(cuda)
            xs[r].C[r * xs[r].S:(r + 1) * xs[r].S].copy_(sl)
            slices.append(sl.cpu().numpy())
        for r in range(world):
            be.p2p_allgather_push(xs[r])
        for r in range(world):
            be.p2p_allgather_wait(xs[r], epoch)
        torch.cuda.synchronize()
        full = np.vstack(slices)
        for r in range(world):
            assert np.array_equal(xs[r].C.cpu().numpy(), full)
    assert all(int(x.status.item()) == 0 for x in xs)


@pytest.mark.timeout(600)
def test_p2p_driver_guard_fallback_rerun(cuda, tmp_path):
    """A rank-deficient A: the Cholesky-QR2 guard fires inside run(); finish()
    re-runs the factorization with TSQR in every QR, the p2p AᵀX exchange
    carrying on with its next epochs, and warns like the reference."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((600, 3)) @ rng.standard_normal((3, 200))
    mp.spawn(_worker, args=(1, _free_port(), a, 8, 1, 2, str(tmp_path), 1), nprocs=1, join=True)
    part = np.load(os.path.join(tmp_path, "rank0.npz"))
    assert int(part["tsqr"]) == 2          # both QRs of A·P̄ by TSQR in the re-run
    assert int(part["epoch"]) == 1 + 2 * 2  # the init self-check, then 2 AᵀX exchanges per factorization,
    # the run and its re-run
    assert int(part["warn"]) == 3          # every orth site warns
    qg = part["q"]
    assert np.abs(qg.T @ qg - np.eye(qg.shape[1])).max() < 1e-12
