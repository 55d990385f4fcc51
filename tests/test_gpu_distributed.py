"""The row-sharded multi-GPU driver with its REAL device path
(CudaBackend: libpbq's kernels through the C ABI) in 2 and 3 ranks that share
one GPU, over the `gloo` backend.

gloo's collectives are host-mediated (stream sync → host copy → TCP → copy
back), so no rank's kernel ever waits on another rank's kernel: this is safe
on one GPU, unlike NCCL ranks sharing a device.  It exercises everything the
N-GPU bench runs except the NCCL transport itself: the sharded sketch rows,
the chunked AᵀX GEMMs with their asynchronous allreduces, the distributed
Cholesky-QR2 of A·P̄ (pbq_cholqr2_dist stages around two Gram allreduces) and
its TSQR fallback, the flag reduction, and the replicated second stage."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, a, d, q, seed, reorth, outdir, chunks, dist_qr):
    import sys
    import warnings

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2103_07245_b200 import device as D
    from paper_2103_07245_b200.distributed import DistributedPbpQlp, shard_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    junk = torch.full((32 << 20,), float("nan"), dtype=torch.float64, device=dev)  # dirty cached memory
    del junk
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, n2 = a.shape
        rows = shard_rows(n1, world)
        run = DistributedPbpQlp(n1, n2, d, q, rows, device=dev, reorthonormalize=reorth, chunks=chunks,
                                dist_qr=dist_qr)
        a_loc = D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(a[rows[rank]:rows[rank + 1]])).to(dev))
        launches0 = run.be.ctx.launch_count
        run.run(a_loc, seed=seed)
        with warnings.catch_warnings(record=True) as rec:
            warnings.simplefilter("always")
            run.finish()
        qg, l, p, r = (t.cpu().numpy() for t in run.factors())
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), q=qg, l=l, p=p, r=r, phi=run.PHI.cpu().numpy(),
                 warn=len(rec), launches=run.be.ctx.launch_count - launches0, tsqr=run.tsqr_fallbacks, orthfb=run.orth_fallbacks)
    finally:
        dist.destroy_process_group()


def _run(a, d, q, seed, reorth, tmp_path, world, chunks=None, dist_qr="auto"):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, a, d, q, seed, reorth, str(tmp_path), chunks, dist_qr), nprocs=world,
             join=True)
    return [np.load(os.path.join(tmp_path, f"rank{g}.npz")) for g in range(world)]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,q,reorth,chunks,dist_qr", [(2, 1, True, None, "auto"), (3, 1, True, 3, "auto"),
                                                           (2, 2, False, None, "auto"), (2, 0, True, 1, "auto"),
                                                           (2, 1, True, None, "tsqr"), (3, 2, True, None, "tsqr")])
def test_sharded_device_path_matches_oracle(cuda, tmp_path, world, q, reorth, chunks, dist_qr):
    """dist_qr "auto": qr(A·P̄) by the distributed Cholesky-QR2 (two d×d
    allreduces); "tsqr": the TSQR tree it falls back to."""
    from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp

    rng = np.random.default_rng(17)
    n1, n2, d = 1500, 700, 48
    a = rng.standard_normal((n1, 60)) @ rng.standard_normal((60, n2)) / 8 + 1e-3 * rng.standard_normal((n1, n2))
    parts = _run(a, d, q, 9, reorth, tmp_path, world, chunks, dist_qr)
    assert all(int(p["tsqr"]) == 0 for p in parts)
    ref = oracle_pbp_qlp(a, d, q=q, seed=9, reorthonormalize=reorth)
    assert all(int(p["launches"]) > 0 for p in parts)  # the device kernels ran in every rank
    phi = np.vstack([p["phi"] for p in parts])
    assert np.array_equal(phi, ref["phi"])  # device sketch: bit-exact
    for p in parts[1:]:  # replicated factors are bitwise identical across ranks
        for k in ("l", "p", "r"):
            assert np.array_equal(p[k], parts[0][k])
    qfull = np.vstack([p["q"] for p in parts])
    tol = conditioning_tolerance(ref["l"], strict=1e-10)
    assert np.all(column_relative_error(qfull, ref["q"]) <= tol)
    assert np.all(column_relative_error(parts[0]["p"], ref["p"]) <= tol)
    lref = np.abs(np.diag(ref["l"]))
    assert np.all(np.abs(np.diag(parts[0]["l"]) - lref) / lref <= conditioning_tolerance(ref["l"], 1e-10, 16.0))
    recon = np.linalg.norm(a - qfull @ parts[0]["l"] @ parts[0]["p"].T) / np.linalg.norm(a)
    ref_recon = np.linalg.norm(a - ref["q"] @ ref["l"] @ ref["p"].T) / np.linalg.norm(a)
    assert abs(recon - ref_recon) <= 1e-10


@pytest.mark.timeout(600)
def test_sharded_device_path_rank_warnings(cuda, tmp_path):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((600, 3)) @ rng.standard_normal((3, 200))
    parts = _run(a, 8, 1, 2, True, tmp_path, 2)
    assert all(int(p["warn"]) == 3 for p in parts)  # every orth site warns on every rank
    assert all(int(p["tsqr"]) == 2 for p in parts)
    assert all(int(p["orthfb"]) == 2 for p in parts)  # ... and both orth(C) calls to the replicated QR  # the Cholesky guard handed both QRs of A·P̄ to TSQR
