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

The workers belong to a :class:`MultiGpuPool`.  ``pbp_qlp_multi_gpu`` starts
one for the call and stops it afterwards: ≈ 3 s of process start-up
(importing torch, creating the CUDA contexts and the process group) before
the first kernel.  A caller with many matrices keeps a pool open and calls
``pool.pbp_qlp`` — or, for peak throughput, runs one process per GPU itself
(``torchrun`` with :class:`DistributedPbpQlp`, A already sharded, as
``bench.py --gpus N`` does), which also avoids handing A over through a host
file per call.
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

__all__ = ["pbp_qlp_multi_gpu", "MultiGpuPool", "usable_world"]

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


def _run_task(rank, world, dev, exchange, task, cache):
    """One factorization in rank ``rank`` (the sharded driver on this rank's rows)."""
    from . import device as D
    from .distributed import DistributedPbpQlp, shard_rows

    root, (n1, n2), d, q, seed, reorth = task
    x = _Exchange(root, n1, n2, d, q, world)
    try:
        rows = shard_rows(n1, world)
        r0, r1 = rows[rank], rows[rank + 1]
        key = (n1, n2, d, q, reorth)
        run = cache.pop(key, None)  # buffers, workspaces and exchange state of this shape (most recent two kept)
        if run is None:
            run = DistributedPbpQlp(n1, n2, d, q, rows, device=dev, reorthonormalize=reorth, exchange=exchange)
        cache[key] = run
        while len(cache) > 2:
            cache.pop(next(iter(cache)))
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
        # recorded for the parent, then re-raised: a rank that fails must take the
        # job down (the parent terminates the others) instead of leaving them in a collective
        x.status[rank, 0] = _DEVICE if isinstance(exc, _exc.DeviceError) else _OTHER
        x.put_message(rank, f"{type(exc).__name__}: {exc}")
        raise
    finally:
        for m in (x.q, x.phi, x.l, x.p, x.r, x.status, x.msg):
            m.flush()


def _pool_worker(rank, world, port, devices, backend, exchange, task_q, result_q):
    """Rank ``rank``: joins the process group once, then serves factorizations
    until it receives ``None``."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", devices[rank])
    torch.cuda.set_device(dev)
    dist.init_process_group(backend, rank=rank, world_size=world)
    result_q.put((rank, "ready"))
    cache = {}
    try:
        while True:
            task = task_q.get()
            if task is None:
                break
            try:
                _run_task(rank, world, dev, exchange, task, cache)
                result_q.put((rank, "done"))
            except Exception:  # noqa: BLE001  already recorded in the status block
                result_q.put((rank, "failed"))
                raise
    finally:
        cache.clear()
        dist.destroy_process_group()


class MultiGpuPool:
    """One worker process per GPU, kept alive across factorizations.

    ``pool.pbp_qlp(a, d, q, seed, reorthonormalize)`` has the arguments,
    errors, warnings and result of :func:`pbp_qlp`; the workers (their CUDA
    contexts, the NCCL communicator, the sharded driver's buffers per shape)
    are started once — seconds — and reused.  Use as a context manager or call
    :meth:`close`.  After a rank fails, the pool is closed and every later
    call raises :class:`DeviceError`.  The workers are started with the
    ``spawn`` method (CUDA cannot be forked): a script that creates a pool at
    import time must do so under ``if __name__ == "__main__":``.
    """

    def __init__(self, devices=None, backend="nccl", exchange="nccl", start_timeout_s=300.0):
        import torch.multiprocessing as mp

        if backend not in ("nccl", "gloo"):
            raise _exc.ParameterError("backend must be 'nccl' or 'gloo'")
        if not torch.cuda.is_available():
            raise _exc.DeviceError("no CUDA device is available; the PbP-QLP path runs only on the GPU")
        if devices is None:
            devices = list(range(torch.cuda.device_count()))
        self.devices = [int(x) for x in devices]
        if not self.devices:
            raise _exc.ParameterError("devices must name at least one GPU")
        if backend == "nccl" and len(set(self.devices)) != len(self.devices):
            raise _exc.ParameterError("the nccl backend needs one distinct GPU per rank")
        self.world = len(self.devices)
        self.backend, self.exchange = backend, exchange
        self.broken = None
        self.procs, self.task_qs = [], []
        if self.world == 1:
            return  # one GPU: calls run pbp_qlp in this process
        ctx = mp.get_context("spawn")
        self.result_q = ctx.Queue()
        port = _free_port()
        for rank in range(self.world):
            tq = ctx.Queue()
            p = ctx.Process(target=_pool_worker, daemon=True,
                            args=(rank, self.world, port, self.devices, backend, exchange, tq, self.result_q))
            p.start()
            self.procs.append(p)
            self.task_qs.append(tq)
        try:
            self._collect("ready", start_timeout_s)
        except Exception:
            self.close()
            raise

    # -- plumbing -------------------------------------------------------------
    def _collect(self, what, timeout_s=None):
        """Wait until every rank reported ``what``; a dead or failed rank raises."""
        import queue
        import time

        seen = set()
        deadline = None if timeout_s is None else time.monotonic() + timeout_s
        while len(seen) < self.world:
            try:
                rank, msg = self.result_q.get(timeout=0.2)
            except queue.Empty:
                dead = [r for r, p in enumerate(self.procs) if not p.is_alive() and r not in seen]
                if dead:
                    raise _exc.DeviceError(f"multi-GPU PbP-QLP: rank {dead[0]} exited (code {self.procs[dead[0]].exitcode})")
                if deadline is not None and time.monotonic() > deadline:
                    raise _exc.DeviceError(f"multi-GPU PbP-QLP: ranks did not report '{what}' within {timeout_s:.0f} s")
                continue
            if msg == "failed":
                raise _exc.DeviceError(f"multi-GPU PbP-QLP: rank {rank} failed")
            if msg == what:
                seen.add(rank)

    def close(self):
        """Stop the workers (idempotent)."""
        for tq in self.task_qs:
            try:
                tq.put(None)
            except Exception:  # noqa: BLE001
                pass
        for p in self.procs:
            p.join(timeout=10 if self.broken is None else 0.5)
            if p.is_alive():
                p.terminate()
                p.join(timeout=5)
        self.procs, self.task_qs = [], []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    # -- the call -------------------------------------------------------------
    def pbp_qlp(self, a, d, q=0, seed=0, reorthonormalize=True):
        """PbP-QLP of the host matrix ``a``, row-sharded over the pool's GPUs."""
        if self.broken:
            raise _exc.DeviceError(f"multi-GPU pool unusable after an earlier failure ({self.broken}); create a new one")
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
        world = self.world
        if usable_world(n1, d, world) < world or world == 1:
            # too short for every rank to hold d rows (or a single GPU): the single-GPU path, in this process
            return pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize,
                           device=torch.device("cuda", self.devices[0]))
        host = ha.host_tensor()
        if host is None:  # a device tensor: the ranks read their rows from host memory
            host = ha.to_device(torch.device("cuda", self.devices[0])).cpu()
        import shutil

        root = _scratch_dir(8 * (n1 * n2 + 2 * n1 * d + n2 * d + 2 * d * d))
        try:
            x = _Exchange(root, n1, n2, d, q, world, create=True)
            x.a[:] = host.numpy()
            x.status[:] = -1
            x.a.flush()
            x.status.flush()
            task = (root, (n1, n2), d, q, seed, bool(reorthonormalize))
            for tq in self.task_qs:
                tq.put(task)
            try:
                self._collect("done")
            except _exc.DeviceError as exc:
                bad = [r for r in range(world) if int(x.status[r, 0]) not in (_OK, _NONFINITE, -1)]
                why = x.message(bad[0]) if bad else str(exc)
                self.broken = why
                self.close()
                raise _exc.DeviceError(f"multi-GPU PbP-QLP: rank {bad[0] if bad else '?'} failed ({why})") from exc
            codes = [int(c) for c in x.status[:, 0]]
            if any(c == _NONFINITE for c in codes):
                raise _exc.MatrixInputError("a contains non-finite entries")
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
    A one-shot :class:`MultiGpuPool`: the workers are started for this call
    and stopped after it.
    """
    ha = HostMatrix(a, "a")
    n1, n2 = ha.shape
    try:
        dd, qq = check_sketch_params(d, q, min(n1, n2))
    except _exc.ParameterError:
        if not ha.all_finite():  # the reference validates A (finiteness included) before d and q
            raise _exc.MatrixInputError("a contains non-finite entries") from None
        raise
    try:
        check_seed(seed)
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
    world = usable_world(n1, dd, len(devices))
    if world == 1:
        return pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize, device=torch.device("cuda", devices[0]))
    with MultiGpuPool(devices[:world], backend, exchange) as pool:
        return pool.pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize)
