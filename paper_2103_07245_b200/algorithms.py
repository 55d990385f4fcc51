"""PbP-QLP on the GPU: the drop-in for ``pbpqlp.pbp_qlp``.

Reference: ``pbp_qlp(a, d, q=0, seed=0, reorthonormalize=True) -> QlpFactors``
(/root/reference/pkg/src/pbpqlp/algorithms.py:209-260), the paper's
Algorithm 3:

1. Φ = gaussian_matrix(n1, d, seed)           (device Philox + ziggurat)
2. C = AᵀΦ ; P̄ = orth(C) ; q × [P̄ = orth(A P̄) ; P̄ = orth(Aᵀ P̄)]
3. D = A P̄ ; (Q, R) = qr(D)
4. (W, R̃) = qr(Rᵀ) ; L = tril(R̃ᵀ) ; P = P̄ W

Everything from step 1 on runs inside one ``pbq_pbp_qlp`` call of libpbq
(include/pbq.h): FP64 DMMA GEMMs and the cooperative Householder QR kernel.
The host only validates, stages A, launches, and reads back one status word
plus the per-``orth`` rank flags (one device→host sync per call).
"""
import ctypes
from dataclasses import dataclass
from typing import Any, Optional

import numpy as np
import torch

from . import _lib
from . import device as _dev
from . import exceptions as _exc
from .linalg import HostMatrix, from_device, householder_qr, to_device_matrix, warn_rank
from .validation import check_index_range, check_seed, check_sketch_params

__all__ = ["SketchRecord", "QlpFactors", "PbpQlpPlan", "pbp_qlp", "pbp_qlp_flops", "pbp_qlp_bytes", "clear_plan_cache"]


class SketchRecord:
    """Provenance of one factorization (algorithms.py:59-72).

    ``test_matrix`` is the Gaussian sketch Φ.  For numpy callers it is copied
    from the device on first access (config 4's Φ is 819 MB).
    """

    __slots__ = ("_phi", "_kind", "_home", "_host", "seed", "d", "q", "passes_over_a")

    def __init__(self, phi, kind, seed, d, q, passes_over_a, home=None):
        self._phi = phi
        self._kind = kind
        self._home = home
        self._host = None
        self.seed = seed
        self.d = d
        self.q = q
        self.passes_over_a = passes_over_a

    @property
    def test_matrix(self):
        if self._host is None:
            self._host = from_device(self._phi, self._kind, self._home)
        return self._host

    @property
    def device_test_matrix(self):
        return self._phi

    def __repr__(self):
        return f"SketchRecord(seed={self.seed}, d={self.d}, q={self.q}, passes_over_a={self.passes_over_a})"


def _diag(x):
    return x.diagonal().clone() if isinstance(x, torch.Tensor) else np.diagonal(x).copy()


@dataclass(frozen=True)
class QlpFactors:
    """``A ≈ q_basis @ l @ p_basis.T`` (algorithms.py:75-128)."""

    q_basis: Any
    l: Any
    p_basis: Any
    first_stage_r: Any
    sketch: Optional[SketchRecord] = None

    @property
    def l_values(self):
        return _diag(self.l)

    @property
    def r_values(self):
        d = _diag(self.first_stage_r)
        return d.abs() if isinstance(d, torch.Tensor) else np.abs(d)

    def approx(self, rank=None):
        if rank is None:
            return self.q_basis @ self.l @ self.p_basis.T
        rank = check_index_range(rank, "rank", 1, self.l.shape[0])
        return self.q_basis[:, :rank] @ self.l[:rank, :rank] @ self.p_basis[:, :rank].T

    def r_blocks(self, k):
        k = check_index_range(k, "k", 1, self.first_stage_r.shape[0] - 1)
        r = self.first_stage_r
        return r[:k, :k], r[:k, k:], r[k:, k:]

    def l_blocks(self, k):
        k = check_index_range(k, "k", 1, self.l.shape[0] - 1)
        l = self.l
        return l[:k, :k], l[k:, :k], l[k:, k:]

    def projection_basis(self):
        w = householder_qr(self.first_stage_r.T).q
        return self.p_basis @ w.T

    def frobenius_error(self, a, rank=None):
        """‖a − approx(rank)‖_F on the GPU in one pass over ``a`` (the
        ``frobenius_error`` of error_curve, analysis.py:238-244)."""
        return residual_norms(a, self, rank)[0]


def residual_norms(a, factors, rank=None, *, device=None):
    """(‖A − Q_k·L_k·P_kᵀ‖_F, ‖A‖_F) for QLP factors truncated to ``rank``
    (QlpFactors.approx, algorithms.py:101-106; for SVD-type factors
    u_k·diag(s_k)·v_kᵀ, analysis.py:182-186), computed by libpbq's fused
    residual GEMM: one pass over A, the n1×n2 approximation is never formed
    (SURVEY.md §8 f2).  ``a`` is validated like the reference's check_matrix."""
    import math

    if hasattr(factors, "l"):  # QLP: Q L Pᵀ
        left, mid, right = factors.q_basis, factors.l, factors.p_basis
    elif hasattr(factors, "t"):  # UTV (cor_utv): U T Vᵀ, T k×d upper trapezoidal
        left, mid, right = factors.u, factors.t, factors.v
    else:  # SVD-type (RsvdFactors): u diag(s) vᵀ
        left, mid, right = factors.u, None, factors.v
    kmax = left.shape[1] if mid is None else mid.shape[0]
    k = kmax if rank is None else check_index_range(rank, "rank", 1, kmax)
    _, a_dev, _, _ = to_device_matrix(a, "a", device)
    dev = a_dev.device
    n1, n2 = a_dev.shape
    if left.shape[0] != n1 or right.shape[0] != n2:
        raise _exc.DimensionError(
            f"factors of a {left.shape[0]}x{right.shape[0]} matrix do not fit a of shape {tuple(a_dev.shape)}"
        )

    def on_dev(x):
        return torch.as_tensor(x).to(device=dev, dtype=torch.float64)

    q = on_dev(left)[:, :k]
    l = on_dev(mid)[:k, :k] if mid is not None else torch.diag(on_dev(factors.s)[:k])
    p = on_dev(right)[:, :k]
    if mid is not None and rank is None and mid.shape[1] > mid.shape[0]:
        # wide UTV core (d > n1): U·T is n1×d, the middle factor the identity
        ctx = _dev.context(dev)
        q = _dev.gemm(ctx, on_dev(left), _dev.as_kernel_operand(on_dev(mid)), trans_a=False)
        l = torch.eye(mid.shape[1], dtype=torch.float64, device=dev)
        p = on_dev(right)
    out = _dev.residual_fro(_dev.context(dev), a_dev, q, l, p)
    r2, a2 = out.tolist()
    return math.sqrt(r2), math.sqrt(a2)


def reconstruction_error(a, factors, rank=None, *, device=None):
    """‖A − approx(rank)‖_F / ‖A‖_F (the north-star reconstruction check)."""
    r, na = residual_norms(a, factors, rank, device=device)
    return r / na if na > 0 else r


def qr_flops(m, d):
    """LAPACK geqrf + orgqr thin-Q flop count, 4md² − 4d³/3."""
    return 4.0 * m * d * d - 4.0 * d ** 3 / 3.0


def pbp_qlp_flops(n1, n2, d, q, reorthonormalize=True):
    """Algorithmic FLOPs of one call."""
    f = (2 * q + 2) * 2.0 * n1 * n2 * d
    if reorthonormalize:
        f += (q + 1) * qr_flops(n2, d) + q * qr_flops(n1, d)
    else:
        f += qr_flops(n2, d)
    f += qr_flops(n1, d) + 8.0 * d ** 3 / 3.0 + 2.0 * n2 * d * d
    return f


def pbp_qlp_bytes(n1, n2, q):
    """Algorithmic HBM bytes: A streamed once per pass."""
    return (2 * q + 2) * 8.0 * n1 * n2


class PbpQlpPlan:
    """Preallocated single-device PbP-QLP for one problem shape.

    ``run`` only enqueues work on the current stream (no host sync), so
    repeated calls can be timed back to back or captured; ``finish`` performs
    the one device→host read of the status/rank flags, raises / warns exactly
    like the reference, and returns the factors as torch tensors.
    """

    def __init__(self, n1, n2, d, q=0, reorthonormalize=True, device=None, explicit_phi=False):
        dev = _dev.require_cuda(device)
        self.n1, self.n2, self.d, self.q = int(n1), int(n2), int(d), int(q)
        self.reorthonormalize = bool(reorthonormalize)
        self.device = dev
        self.ctx = _dev.context(dev)
        self.Q = _dev.empty_matrix(n1, d, dev)
        self.P = _dev.empty_matrix(n2, d, dev)
        self.L = _dev.empty_matrix(d, d, dev)
        self.R = _dev.empty_matrix(d, d, dev)
        self.PHI = None if explicit_phi else _dev.empty_matrix(n1, d, dev)
        self.flags = torch.zeros(2 * q + 2, dtype=torch.int32, device=dev)  # [status bits, rank flags...]
        self.prob = _lib.PbqProblem()
        self.prob.n1, self.prob.n2, self.prob.d, self.prob.q = n1, n2, d, q
        self.prob.reorthonormalize = 1 if reorthonormalize else 0
        self.prob.check_finite = 1
        self.out = _lib.PbqOutputs()
        o = self.out
        o.q, o.ldq = self.Q.data_ptr(), self.Q.stride(0)
        o.l, o.ldl = self.L.data_ptr(), self.L.stride(0)
        o.p, o.ldp = self.P.data_ptr(), self.P.stride(0)
        o.r, o.ldr = self.R.data_ptr(), self.R.stride(0)
        if self.PHI is not None:
            o.phi, o.ldphi = self.PHI.data_ptr(), self.PHI.stride(0)
        o.nonfinite = self.flags.data_ptr()
        o.rank_flags = self.flags.data_ptr() + 4
        if explicit_phi:
            self.prob.phi = 1  # sizing only: explicit sketch needs no generator workspace
        nbytes = ctypes.c_size_t()
        self.ctx.check(self.ctx.lib.pbq_pbp_qlp_workspace_bytes(self.ctx.handle, ctypes.byref(self.prob),
                                                               ctypes.byref(nbytes)), "pbp_qlp workspace")
        self.ws_bytes = nbytes.value
        self.ws = _dev.workspace(self.ws_bytes, dev)
        self.seed = 0
        self.phi_in = None

    def run_streamed(self, host, seed=0, chunks=16):
        """Factor a host (CPU) float64 tensor, streaming it to the device in
        row chunks on a copy stream while the first pass C = AᵀΦ accumulates
        chunk by chunk on the compute stream (β = 1 GEMM updates); the rest of
        the pipeline starts from that C.  Returns the device copy of A.

        Pinned input is copied by DMA straight from its pages.  Pageable
        input (numpy arrays) goes through a ring of STAGE_SLOTS pinned
        staging buffers: the host copies chunk i+1 into a free slot (torch's
        multithreaded CPU copy) while the DMA engine moves chunk i, so the
        link and host memory bandwidth overlap instead of the runtime's
        synchronous pageable path (~10 GB/s)."""
        dev = self.device
        if tuple(host.shape) != (self.n1, self.n2):
            raise _exc.DimensionError(f"plan is for {(self.n1, self.n2)}, got {tuple(host.shape)}")
        seed = check_seed(seed)
        self.seed = seed
        self.prob.seed_dev = None
        if self.PHI is None:
            raise _exc.ParameterError("plan was built for an explicit sketch")
        if getattr(self, "A_dev", None) is None:
            self.A_dev = _dev.empty_matrix(self.n1, self.n2, dev)
            self.C0 = _dev.empty_matrix(self.n2, self.d, dev)
            self.copy_stream = torch.cuda.Stream(dev)
        A, C0 = self.A_dev, self.C0
        compute = torch.cuda.current_stream(dev)
        self.copy_stream.wait_stream(compute)  # A may still be read by a previous call
        self.flags.zero_()
        self.sk_status = getattr(self, "sk_status", None)
        if self.sk_status is None:
            self.sk_status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.sk_status.zero_()
        _dev.gaussian(self.ctx, self.n1, self.d, seed, dev, out=self.PHI, status=self.sk_status)
        nchunks = max(1, min(int(chunks), self.n1 // max(self.d, 1)))
        bounds = [(self.n1 * i) // nchunks for i in range(nchunks + 1)]
        pinned = host.is_pinned()
        if not pinned:
            rows_max = max(bounds[i + 1] - bounds[i] for i in range(nchunks))
            ring = getattr(self, "stage", None)
            if ring is None or ring[0].shape[0] < rows_max:
                # pinned staging ring, kept with the plan (pinned allocations are slow)
                self.stage = ring = [torch.empty((rows_max, self.n2), dtype=torch.float64, pin_memory=True)
                                     for _ in range(STAGE_SLOTS)]
                self.stage_ev = [None] * STAGE_SLOTS
        for i in range(nchunks):
            r0, r1 = bounds[i], bounds[i + 1]
            if pinned:
                src = host[r0:r1]
            else:
                k = i % STAGE_SLOTS
                if self.stage_ev[k] is not None:
                    self.stage_ev[k].synchronize()  # the DMA out of this slot has finished
                src = ring[k][:r1 - r0]
                src.copy_(host[r0:r1])
            with torch.cuda.stream(self.copy_stream):
                A[r0:r1].copy_(src, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            if not pinned:
                self.stage_ev[k] = ev
            compute.wait_event(ev)
            _dev.gemm(self.ctx, A[r0:r1], self.PHI[r0:r1], trans_a=True, out=C0, beta=0.0 if i == 0 else 1.0,
                      nonfinite=self.flags[0:1])
        self.prob.c_init, self.prob.ldc_init = C0.data_ptr(), C0.stride(0)
        self.prob.phi, self.prob.ldphi = self.PHI.data_ptr(), self.PHI.stride(0)
        self.prob.a, self.prob.lda = A.data_ptr(), A.stride(0)
        self.prob.seed_lo, self.prob.seed_hi = seed & ((1 << 64) - 1), seed >> 64
        self.phi_in = None
        with self.ctx.lock:
            st = self.ctx.lib.pbq_pbp_qlp(self.ctx.handle, ctypes.byref(self.prob), ctypes.byref(self.out),
                                          _dev.ptr(self.ws), self.ws_bytes, _dev.stream_ptr(dev))
            self.ctx.check(st, "pbp_qlp")
        self.prob.c_init, self.prob.ldc_init = None, 0
        self._streamed = True
        return A

    def detach_sketch(self):
        """Hand the seeded sketch buffer to the caller (a SketchRecord) and
        give the plan a fresh one, so a cached plan's next call cannot
        overwrite a returned Φ."""
        phi = self.PHI
        if phi is not None:
            self.PHI = _dev.empty_matrix(self.n1, self.d, self.device)
            self.out.phi, self.out.ldphi = self.PHI.data_ptr(), self.PHI.stride(0)
        return phi

    def run(self, A, seed=0, phi=None, _seed_dev=None):
        """Enqueue one factorization of the kernel-ready device matrix ``A``."""
        self.prob.seed_dev = _seed_dev  # set only while ``capture`` records the graph
        if tuple(A.shape) != (self.n1, self.n2):
            raise _exc.DimensionError(f"plan is for {(self.n1, self.n2)}, got {tuple(A.shape)}")
        seed = check_seed(seed)
        self.seed = seed
        self.prob.a, self.prob.lda = A.data_ptr(), A.stride(0)
        self.prob.seed_lo, self.prob.seed_hi = seed & ((1 << 64) - 1), seed >> 64
        if phi is not None:
            if tuple(phi.shape) != (self.n1, self.d):
                raise _exc.DimensionError(f"phi must have shape ({self.n1}, {self.d}), got {tuple(phi.shape)}")
            self.prob.phi, self.prob.ldphi = phi.data_ptr(), phi.stride(0)
        else:
            if self.PHI is None:
                raise _exc.ParameterError("plan was built for an explicit sketch; pass phi")
            self.prob.phi, self.prob.ldphi = None, 0
        self.phi_in = phi
        self._streamed = False
        with self.ctx.lock:
            st = self.ctx.lib.pbq_pbp_qlp(self.ctx.handle, ctypes.byref(self.prob), ctypes.byref(self.out),
                                          _dev.ptr(self.ws), self.ws_bytes, _dev.stream_ptr(self.device))
            self.ctx.check(st, "pbp_qlp")

    # -- CUDA graph of the whole pipeline -----------------------------------
    def capture(self, A):
        """Capture one factorization of the device matrix ``A`` (seeded mode)
        into a CUDA graph; ``replay(seed)`` then re-runs all of it — sketch,
        every pass and QR — with one graph launch.  The sketch reads its key
        from device memory (``pbq_problem.seed_dev``), so each replay can use a
        new seed; ``A`` and the outputs are the captured buffers."""
        if self.PHI is None:
            raise _exc.ParameterError("capture needs a plan with a seeded sketch")
        dev = self.device
        self.seed_dev = torch.zeros(2, dtype=torch.int64, device=dev)
        self.run(A, seed=0)  # warm: tables, function attributes, lazy module loads
        launches0 = self.ctx.launch_count
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            self.run(A, seed=0, _seed_dev=self.seed_dev.data_ptr())
        self.prob.seed_dev = None
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph_launches = self.ctx.launch_count - launches0  # kernels per replay
        self.graph, self.graph_A = graph, A
        return graph

    def replay(self, seed=0):
        """Launch the captured factorization with sketch seed ``seed``."""
        seed = check_seed(seed)
        self.seed = seed
        lo, hi = seed & ((1 << 64) - 1), seed >> 64
        to_i64 = lambda v: v - (1 << 64) if v >= (1 << 63) else v  # noqa: E731  (same 64 bits)
        self.seed_dev[0].fill_(to_i64(lo))
        self.seed_dev[1].fill_(to_i64(hi))
        self.phi_in = None
        self._streamed = False
        self.graph.replay()

    def finish(self, stacklevel=3):
        fl = self.flags.cpu().tolist()  # the one device→host synchronisation
        if getattr(self, "_streamed", False) and int(self.sk_status.item()):
            fl[0] |= 2
        if fl[0] & 1:
            raise _exc.MatrixInputError("a contains non-finite entries")
        if fl[0] & 2:
            raise _exc.DeviceError("sketch generator overflow (internal error)")
        for flag in fl[1:]:
            warn_rank(flag, stacklevel=stacklevel + 1)
        return fl


#: host inputs at least this large stream to the GPU in row chunks overlapped
#: with the first pass (PbpQlpPlan.run_streamed)
STREAM_MIN_BYTES = 64 << 20
#: pinned staging buffers in the pageable-input ring of run_streamed
STAGE_SLOTS = 3

# Plans of recent host-input calls, keyed by device and problem shape: a plan
# holds the device copy of A, the factor buffers, the workspace and the
# pinned staging ring, so a repeated call of the same shape (the reference's
# runtime protocol, an estimator refit) allocates nothing.  Only calls whose
# results are copied back to the host use it (device callers get tensors
# that alias the plan's buffers).  A plan is checked out while in use, so
# concurrent calls never share one.  PBQ_PLAN_CACHE=0 disables it.
_PLAN_CACHE = {}
_PLAN_CACHE_MAX = 2
_PLAN_LOCK = __import__("threading").Lock()


def _plan_cache_enabled():
    import os

    return os.environ.get("PBQ_PLAN_CACHE", "1") != "0"


def _checkout_plan(n1, n2, d, q, reorth, dev):
    key = (torch.device(dev).index, n1, n2, d, q, bool(reorth))
    if _plan_cache_enabled():
        with _PLAN_LOCK:
            plan = _PLAN_CACHE.pop(key, None)
        if plan is not None:
            return key, plan
    return key, PbpQlpPlan(n1, n2, d, q, reorth, dev)


def _checkin_plan(key, plan):
    if not _plan_cache_enabled():
        return
    with _PLAN_LOCK:
        _PLAN_CACHE[key] = plan
        while len(_PLAN_CACHE) > _PLAN_CACHE_MAX:
            _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))


def clear_plan_cache():
    """Release the cached host-input plans (device memory of A and the factors)
    and the pinned staging rings of host-array copies."""
    with _PLAN_LOCK:
        _PLAN_CACHE.clear()
    _dev.release_staging()


def _to_host(t, kind, home):
    """Device result → caller type, through a pinned buffer for host callers."""
    if kind == "torch" and home is not None and torch.device(home).type == "cuda":
        return from_device(t, kind, home)
    buf = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    buf.copy_(t, non_blocking=True)
    return buf


def pbp_qlp(a, d, q=0, seed=0, reorthonormalize=True, *, phi=None, device=None):
    """Projection-based partial QLP factorization of ``a`` on the GPU.

    Same signature, arguments, errors, warnings and return fields as the
    reference (algorithms.py:209-260).  Extensions (keyword-only):
    ``phi`` supplies the sketch explicitly (oracle mode, n1×d); ``device``
    picks the GPU for array-like inputs.  numpy/array-like input returns numpy
    factors; a torch tensor returns torch tensors on the tensor's home device.
    Large host inputs are streamed to the GPU in row chunks while the first
    pass over A runs (PbpQlpPlan.run_streamed).
    """
    ha = HostMatrix(a, "a")
    n1, n2 = ha.shape
    try:
        d, q = check_sketch_params(d, q, min(n1, n2))
    except _exc.ParameterError:
        # the reference validates A (including finiteness) before d and q
        if not ha.all_finite():
            raise _exc.MatrixInputError("a contains non-finite entries") from None
        raise
    try:
        seed = check_seed(seed)
    except ValueError:
        # likewise for the seed (numpy's Philox rejects it only after
        # check_matrix has scanned A, algorithms.py:239-242)
        if not ha.all_finite():
            raise _exc.MatrixInputError("a contains non-finite entries") from None
        raise
    kind, home = ha.kind, ha.home
    host = ha.host_tensor()
    streamed = host is not None and phi is None and n1 * n2 * 8 >= STREAM_MIN_BYTES and n1 >= 2 * d
    host_side = not (kind == "torch" and home is not None and torch.device(home).type == "cuda")
    key = None
    if streamed:
        dev = _dev.require_cuda(device)
        key, plan = _checkout_plan(n1, n2, d, q, reorthonormalize, dev)
        plan.run_streamed(host, seed)
        PHI = None
    else:
        A = ha.to_device(device)
        dev = A.device
        PHI = None
        if phi is not None:
            _, PHI, _, _ = to_device_matrix(phi, "phi", dev)
        if host_side and phi is None:
            key, plan = _checkout_plan(n1, n2, d, q, reorthonormalize, dev)
        else:
            plan = PbpQlpPlan(n1, n2, d, q, reorthonormalize, dev, explicit_phi=phi is not None)
        plan.run(A, seed, PHI)
    if host_side:
        outs = [_to_host(t, kind, home) for t in (plan.Q, plan.L, plan.P, plan.R)]
    try:
        plan.finish(stacklevel=3)  # synchronises the stream (also completes the copies above)
    finally:
        phi_dev = PHI if PHI is not None else plan.detach_sketch() if key is not None else plan.PHI
        if key is not None:
            _checkin_plan(key, plan)
    if host_side:
        outs = [o.numpy() if kind == "numpy" else o for o in outs]
    else:
        outs = [from_device(t, kind, home) for t in (plan.Q, plan.L, plan.P, plan.R)]
    passes = 2 * q + 2
    sketch = SketchRecord(phi_dev, kind, seed, d, q, passes, home)
    if phi is not None and kind == "numpy":
        sketch._host = np.asarray(phi, dtype=np.float64)
    return QlpFactors(outs[0], outs[1], outs[2], outs[3], sketch)
