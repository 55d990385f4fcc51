"""One call, several GPUs: ``pbp_qlp_multi_gpu(a, d, q, seed, …, devices=…)``.

The reference's ``pbp_qlp`` (algorithms.py:209-260) is a single host call on a
host array.  On a multi-GPU box the same call shape is kept: the launcher
starts one worker process per GPU (the layout ``torch.distributed`` and NCCL
are built for — a context per process, no GIL between the ranks' enqueue
threads), hands every rank its contiguous row block of A through shared
memory, runs the row-sharded driver (:class:`DistributedPbpQlp`, SURVEY.md
§8e) and collects Q (row blocks), L, P, R and Φ back into shared host
buffers.  Arguments, errors, warnings and the returned :class:`QlpFactors`
are those of ``pbp_qlp``.

Every call starts its own workers: seconds of process start-up (importing
torch, creating the CUDA contexts and the NCCL communicator) before the first
kernel, which only a large A amortises.  A service that factors many matrices
keeps one process per GPU alive instead — ``torchrun`` with
:class:`DistributedPbpQlp`, A already sharded, as ``bench.py --gpus N`` does
(its plan objects and CUDA graphs are reused from call to call).
"""
import os
import socket
import warnings

import numpy as np
import torch

from . import exceptions as _exc
from .algorithms import QlpFactors, SketchRecord, pbp_qlp
from .linalg import HostMatrix, warn_rank
from .validation import check_seed, check_sketch_params

__all__ = ["pbp_qlp_multi_gpu", "usable_world"]

# worker status codes written to the shared status block
_OK, _NONFINITE, _DEVICE, _OTHER = 0, 3, 4, 9  # (−1: the rank never reported)


def usable_world(n1, d, ndev):
    """Largest rank count ≤ ndev whose balanced row shards all hold ≥ d rows
    (the sharded QR factors each rank's block on its own first)."""
    world = max(1, int(ndev))
    while world > 1 and n1 // world < d:
        world -= 1
    return world


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _Exchange:
    """The job's host buffers as memory-mapped files in one scratch directory
    (RAM-backed /dev/shm when it has room, else the temp directory): A in, the
    factors, Φ and a status block out.  Workers open the same files."""

    def __init__(self, root, n1, n2, d, q, world, create=False):
        self.root = root
        mode = "w+" if create else "r+"
        mm = lambda name, dtype, shape: np.memmap(os.path.join(root, name), dtype=dtype, mode=mode, shape=shape)  # noqa: E731
        self.a = mm("a", np.float64, (n1, n2))
        self.q = mm("q", np.float64, (n1, d))
        self.phi = mm("phi", np.float64, (n1, d))
        self.l = mm("l", np.float64, (d, d))
        self.p = mm("p", np.float64, (n2, d))
        self.r = mm("r", np.float64, (d, d))
        self.status = mm("status", np.int64, (world, 2 * q + 8))  # [code, finish() flags…] per rank
        self.msg = mm("msg", np.uint8, (world, 512))

    def put_message(self, rank, text):
        raw = text.encode("utf-8", "replace")[:511]
        self.msg[rank, :len(raw)] = np.frombuffer(raw, dtype=np.uint8)
        self.msg[rank, len(raw)] = 0

    def message(self, rank):
        return bytes(self.msg[rank]).split(b"\0", 1)[0].decode("utf-8", "replace")


def _scratch_dir(nbytes):
    import shutil
    import tempfile

    base = None
    try:
        if shutil.disk_usage("/dev/shm").free > 1.1 * nbytes + (64 << 20):
            base = "/dev/shm"
    except OSError:
        pass
    return tempfile.mkdtemp(prefix="pbq_multigpu_", dir=os.environ.get("PBQ_TMPDIR", base))


def _worker(rank, world, port, devices, backend, exchange, root, shape, d, q, seed, reorth):
    """Rank ``rank`` of the job (runs in its own process)."""
    import torch.distributed as dist

    from . import device as D
    from .distributed import DistributedPbpQlp, shard_rows

    n1, n2 = shape
    x = _Exchange(root, n1, n2, d, q, world)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", devices[rank])
    torch.cuda.set_device(dev)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        rows = shard_rows(n1, world)
        r0, r1 = rows[rank], rows[rank + 1]
        run = DistributedPbpQlp(n1, n2, d, q, rows, device=dev, reorthonormalize=reorth, exchange=exchange)
        a_loc = D.empty_matrix(r1 - r0, n2, dev)
        D.h2d(torch.from_numpy(np.ascontiguousarray(x.a[r0:r1])), a_loc)  # pinned staging ring (device.h2d)
        run.run(a_loc, seed=seed)
        with warnings.catch_warnings(record=True):
            warnings.simplefilter("always")  # the parent re-emits them from the flags
            flags = run.finish()
        qg, l, p, r = run.factors()
        x.q[r0:r1] = qg.cpu().numpy()
        x.phi[r0:r1] = run.PHI.cpu().numpy()
        if rank == 0:
            x.l[:] = l.cpu().numpy()
            x.p[:] = p.cpu().numpy()
            x.r[:] = r.cpu().numpy()
            x.status[0, 1:1 + len(flags)] = flags
        x.status[rank, 0] = _OK
    except _exc.MatrixInputError:  # raised by finish() on every rank alike (the flag is allreduced)
        x.status[rank, 0] = _NONFINITE
    except Exception as exc:  # noqa: BLE001
        # recorded for the parent, then re-raised: a rank that dies must take the
        # job down (mp.spawn terminates the others) instead of leaving them in a collective
        x.status[rank, 0] = _DEVICE if isinstance(exc, _exc.DeviceError) else _OTHER
        x.put_message(rank, f"{type(exc).__name__}: {exc}")
        x.status.flush()
        x.msg.flush()
        raise
    finally:
        for m in (x.q, x.phi, x.l, x.p, x.r, x.status, x.msg):
            m.flush()
        dist.destroy_process_group()


def pbp_qlp_multi_gpu(a, d, q=0, seed=0, reorthonormalize=True, *, devices=None, backend="nccl", exchange="nccl"):
    """PbP-QLP of the host matrix ``a`` row-sharded over several GPUs of this node.

    Same arguments, errors, warnings and result as :func:`pbp_qlp`
    (reference algorithms.py:209-260); factors come back as numpy arrays.
    ``devices``: CUDA indices, one rank each (default: every visible GPU;
    ranks are dropped until each holds at least ``d`` rows).  ``backend``:
    ``"nccl"`` (one GPU per rank), or ``"gloo"`` for validation runs whose
    ranks may share a GPU (host-mediated collectives).  ``exchange``: the AᵀX
    exchange of :class:`DistributedPbpQlp` (``"nccl"`` or ``"p2p"``).
    One device, or a matrix too short to shard, runs :func:`pbp_qlp`.
    """
    ha = HostMatrix(a, "a")
    n1, n2 = ha.shape
    try:
        d, q = check_sketch_params(d, q, min(n1, n2))
    except _exc.ParameterError:
        if not ha.all_finite():  # the reference validates A (finiteness included) before d and q
            raise _exc.MatrixInputError("a contains non-finite entries") from None
        raise
    try:
        seed = check_seed(seed)
    except ValueError:
        if not ha.all_finite():
            raise _exc.MatrixInputError("a contains non-finite entries") from None
        raise
    if backend not in ("nccl", "gloo"):
        raise _exc.ParameterError("backend must be 'nccl' or 'gloo'")
    if not torch.cuda.is_available():
        raise _exc.DeviceError("no CUDA device is available; the PbP-QLP path runs only on the GPU")
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [int(x) for x in devices]
    if not devices:
        raise _exc.ParameterError("devices must name at least one GPU")
    if backend == "nccl" and len(set(devices)) != len(devices):
        raise _exc.ParameterError("the nccl backend needs one distinct GPU per rank")
    world = usable_world(n1, d, len(devices))
    devices = devices[:world]
    if world == 1:
        return pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize, device=torch.device("cuda", devices[0]))

    host = ha.host_tensor()
    if host is None:  # a device tensor: the ranks read their rows from host memory
        host = ha.to_device(torch.device("cuda", devices[0])).cpu()
    import shutil

    import torch.multiprocessing as mp

    root = _scratch_dir(8 * (n1 * n2 + 2 * n1 * d + n2 * d + 2 * d * d))
    try:
        x = _Exchange(root, n1, n2, d, q, world, create=True)
        x.a[:] = host.numpy()
        x.status[:] = -1
        x.a.flush()
        x.status.flush()
        try:
            mp.spawn(_worker, args=(world, _free_port(), devices, backend, exchange, root, (n1, n2), d, q, seed,
                                    bool(reorthonormalize)), nprocs=world, join=True)
        except Exception as exc:  # noqa: BLE001  a rank raised or died: report what it recorded
            bad = [r for r in range(world) if int(x.status[r, 0]) not in (_OK, _NONFINITE, -1)]
            why = x.message(bad[0]) if bad else f"{type(exc).__name__}: {str(exc)[:300]}"
            raise _exc.DeviceError(f"multi-GPU PbP-QLP: rank {bad[0] if bad else '?'} failed ({why})") from exc
        codes = [int(c) for c in x.status[:, 0]]
        if any(c == _NONFINITE for c in codes):
            raise _exc.MatrixInputError("a contains non-finite entries")
        for rank, c in enumerate(codes):
            if c != _OK:
                raise _exc.DeviceError(f"multi-GPU PbP-QLP: rank {rank} failed ({x.message(rank) or 'no status'})")
        n_orth = (2 * q + 1) if reorthonormalize else 1
        flags = [int(f) for f in x.status[0, 3:3 + n_orth]]  # finish(): [nonfinite, sketch status, orth flags…]
        outs = [np.array(m) for m in (x.q, x.l, x.p, x.r, x.phi)]  # copies: the files go away below
        del x
    finally:
        shutil.rmtree(root, ignore_errors=True)
    for flag in flags:
        warn_rank(flag, stacklevel=3)
    sketch = SketchRecord(None, "numpy", seed, d, q, 2 * q + 2, None)
    sketch._host = outs[4]
    return QlpFactors(outs[0], outs[1], outs[2], outs[3], sketch)
