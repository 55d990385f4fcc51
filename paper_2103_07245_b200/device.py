"""Per-device library contexts and thin typed wrappers over the C ABI.

PyTorch provides device memory (caching allocator), streams and the NCCL
process group; every FLOP of the PbP-QLP path runs in libpbq's kernels.
Matrices are torch float64 CUDA tensors, row-major, with an even row stride
(the kernels stage 16-byte chunks).
"""
import ctypes
import threading

import torch

from . import _lib
from . import exceptions as _exc

JACOBI_ACCUMULATE = 1  # pbq.h PBQ_JACOBI_ACCUMULATE
JACOBI_PRECONDITION = 2  # pbq.h PBQ_JACOBI_PRECONDITION

_ctx_lock = threading.Lock()
_contexts = {}


class Context:
    """One ``pbq_ctx`` bound to a CUDA device (not thread-safe: guarded)."""

    def __init__(self, device_index):
        self.lib = _lib.load()
        self.device_index = device_index
        self.lock = threading.RLock()
        handle = ctypes.c_void_p()
        st = self.lib.pbq_ctx_create(device_index, ctypes.byref(handle))
        if st != _lib.PBQ_OK:
            raise _exc.DeviceError(f"pbq_ctx_create(device={device_index}) failed with status {st}")
        self.handle = handle

    @property
    def sm_count(self):
        return self.lib.pbq_ctx_sm_count(self.handle)

    @property
    def launch_count(self):
        return int(self.lib.pbq_ctx_launch_count(self.handle))

    def check(self, status, what):
        _lib.raise_status(status, self.handle, what)

    QR_AUTO, QR_HOUSEHOLDER, QR_CHOLQR_NOSERIES, QR_CHOLQR_CHAIN = 0, 1, 2, 3

    def clear_error(self):
        """Reset the CUDA last-error state (after a failed stream capture);
        returns the pending cudaError_t code (0: none)."""
        with self.lock:
            return int(self.lib.pbq_clear_error(self.handle))

    def set_qr_method(self, method):
        """0: Cholesky-QR2 with on-device Householder fallback (default);
        1: Householder kernel only; 2: as 0 with the blocked Cholesky in the
        second pass (test hook)."""
        with self.lock:
            self.check(self.lib.pbq_set_qr_method(self.handle, int(method)), "set_qr_method")

    def set_basis_orth(self, on):
        """True (default): pbp_qlp's intermediate orth calls run basis-only (one
        Cholesky-QR pass); False: every orth is the full QR (A/B switch)."""
        with self.lock:
            self.check(self.lib.pbq_set_basis_orth(self.handle, int(bool(on))), "set_basis_orth")

    def set_p2p_timeout_ms(self, ms):
        """Spin limit of the peer-memory waits launched from now on (default 20 s)."""
        with self.lock:
            self.check(self.lib.pbq_set_p2p_timeout_ms(self.handle, int(ms)), "set_p2p_timeout_ms")

    def cholqr_stats(self, stats):
        """Count [Cholesky-QR completions, Householder fallbacks, series last pass,
        shifted-route completions] into the
        int32 device tensor ``stats`` (None to stop)."""
        with self.lock:
            self.check(self.lib.pbq_debug_cholqr_stats(self.handle, ptr(stats)), "cholqr_stats")

    def profile_begin(self, capacity=4096):
        """Start bracketing every kernel this context enqueues with CUDA events."""
        self.check(self.lib.pbq_profile_begin(self.handle, int(capacity)), "profile_begin")

    def profile_end(self):
        """(ms, launches) per kernel class {gemm, qr, sketch, other} since begin."""
        ms = (ctypes.c_double * 4)()
        n = (ctypes.c_int32 * 4)()
        self.check(self.lib.pbq_profile_end(self.handle, ms, n), "profile_end")
        names = ("gemm", "qr", "sketch", "other")
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise _exc.DeviceError("no CUDA device is available; the PbP-QLP path runs only on the GPU")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise _exc.DeviceError(f"expected a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def context(device):
    dev = require_cuda(device)
    with _ctx_lock:
        ctx = _contexts.get(dev.index)
        if ctx is None:
            with torch.cuda.device(dev):
                ctx = Context(dev.index)
            _contexts[dev.index] = ctx
    return ctx


def stream_ptr(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def even_ld(n):
    return n + (n & 1)


def empty_matrix(rows, cols, device):
    """rows×cols float64 view of a (rows, even_ld(cols)) allocation."""
    ld = even_ld(cols)
    buf = torch.empty((rows, ld), dtype=torch.float64, device=device)
    return buf[:, :cols] if ld != cols else buf


def ld_of(t):
    return t.stride(0)


def as_kernel_operand(t):
    """Return ``t`` or a copy whose layout the kernels accept (row-major,
    unit column stride, even row stride, 16-byte aligned base)."""
    ok = (
        t.dtype == torch.float64
        and t.dim() == 2
        and t.stride(1) == 1
        and t.stride(0) >= t.shape[1]
        and t.stride(0) % 2 == 0
        and t.data_ptr() % 16 == 0
    )
    if ok:
        return t
    out = empty_matrix(t.shape[0], t.shape[1], t.device)
    out.copy_(t)
    return out


# Pinned staging ring for pageable host → device copies (per device; reused
# across calls because pinned allocations are slow).
STAGE_SLOTS = 3
STAGE_CHUNK_BYTES = 64 << 20
_stage_lock = threading.Lock()
_stage = {}


def h2d(host, out):
    """Copy the CPU float64 matrix ``host`` into the device view ``out``.

    Pinned or small inputs take one copy.  A large pageable input (a numpy
    array: the reference's calling convention) goes through a ring of
    STAGE_SLOTS pinned chunk buffers: the host copies chunk i+1 into a free
    slot (torch's multithreaded CPU copy) while the DMA engine moves chunk i,
    instead of the runtime's synchronous pageable path (~10 GB/s).  The copies
    are ordered on the current stream."""
    rows, cols = host.shape
    if host.is_pinned() or rows * cols * 8 < (16 << 20):
        out.copy_(host, non_blocking=host.is_pinned())
        return out
    dev = out.device
    per = max(1, STAGE_CHUNK_BYTES // (8 * cols))
    stream = torch.cuda.current_stream(dev)
    with _stage_lock:
        ring = _stage.get(dev.index)
        if ring is None or ring[0][0].numel() < per * cols:
            ring = ([torch.empty(per * cols, dtype=torch.float64, pin_memory=True) for _ in range(STAGE_SLOTS)],
                    [None] * STAGE_SLOTS)
            _stage[dev.index] = ring
        bufs, evs = ring
        for i, r0 in enumerate(range(0, rows, per)):
            r1 = min(rows, r0 + per)
            k = i % STAGE_SLOTS
            if evs[k] is not None:
                evs[k].synchronize()  # the DMA out of this slot has finished
            b = bufs[k][:(r1 - r0) * cols].view(r1 - r0, cols)
            b.copy_(host[r0:r1])
            out[r0:r1].copy_(b, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            evs[k] = ev
    return out


def release_staging():
    """Free the pinned staging rings of h2d (they are re-created on demand)."""
    with _stage_lock:
        for bufs, evs in _stage.values():
            for ev in evs:
                if ev is not None:
                    ev.synchronize()
        _stage.clear()


def workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


# ---------------------------------------------------------------- kernels --
def gemm(ctx, a, b, trans_a, out=None, alpha=1.0, beta=0.0, nonfinite=None):
    """out = alpha·op(a)·b + beta·out, op = transpose when ``trans_a``."""
    dev = a.device
    a = as_kernel_operand(a)
    b = as_kernel_operand(b)
    if trans_a:
        K, M = a.shape
    else:
        M, K = a.shape
    N = b.shape[1]
    if b.shape[0] != K:
        raise _exc.DimensionError(f"gemm: inner dimensions differ ({K} vs {b.shape[0]})")
    if out is None:
        out = empty_matrix(M, N, dev)
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_gemm_workspace_bytes(ctx.handle, M, N, K, ctypes.byref(nbytes)), "gemm workspace")
        ws = workspace(nbytes.value, dev)
        fn = ctx.lib.pbq_gemm_tn if trans_a else ctx.lib.pbq_gemm_nn
        st = fn(ctx.handle, M, N, K, float(alpha), ptr(a), ld_of(a), ptr(b), ld_of(b), float(beta), ptr(out),
                ld_of(out), ptr(nonfinite), ptr(ws), nbytes.value, stream_ptr(dev))
        ctx.check(st, "gemm")
    return out


# ------------------------------------------------ fused AᵀX exchange (p2p) --
def gemm_tn_scatter(ctx, a, x, xchg, nonfinite=None):
    """C_rank = aᵀ·x with every finished tile stored into its slice owner's
    landing slot through the peer mapping (pbq_gemm_tn_scatter)."""
    a = as_kernel_operand(a)
    x = as_kernel_operand(x)
    K, M = a.shape
    N = x.shape[1]
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_gemm_workspace_bytes(ctx.handle, M, N, K, ctypes.byref(nbytes)), "gemm workspace")
        ws = workspace(nbytes.value, a.device)
        st = ctx.lib.pbq_gemm_tn_scatter(ctx.handle, M, N, K, ptr(a), ld_of(a), ptr(x), ld_of(x), ptr(xchg.land_ptrs),
                                         ptr(xchg.cnt_ptrs), xchg.rank, xchg.world, xchg.S, xchg.ldl, ptr(nonfinite),
                                         ptr(ws), nbytes.value, stream_ptr(a.device))
        ctx.check(st, "gemm_tn_scatter")


def xchg_reduce(ctx, xchg, n2, n, tile_target):
    with ctx.lock:
        st = ctx.lib.pbq_xchg_reduce(ctx.handle, xchg.rank, xchg.world, n2, n, xchg.S, ptr(xchg.land), xchg.ldl,
                                     ptr(xchg.c_ptrs), xchg.ldl, ptr(xchg.cnt), ctypes.c_uint32(tile_target),
                                     ptr(xchg.done_ptrs), stream_ptr(xchg.land.device))
        ctx.check(st, "xchg_reduce")


def xchg_wait(ctx, xchg, done_target):
    with ctx.lock:
        st = ctx.lib.pbq_xchg_wait(ctx.handle, ptr(xchg.done), ctypes.c_uint32(done_target),
                                   stream_ptr(xchg.land.device))
        ctx.check(st, "xchg_wait")


def p2p_push(ctx, src, n, dst_ptrs, slot, rank, world, cnt_ptrs):
    with ctx.lock:
        st = ctx.lib.pbq_p2p_push(ctx.handle, ptr(src), int(n), ptr(dst_ptrs), int(slot), int(rank), int(world),
                                  ptr(cnt_ptrs), stream_ptr(src.device))
        ctx.check(st, "p2p_push")


def p2p_sum(ctx, slots, slot, world, n, out, cnt, target, status):
    with ctx.lock:
        st = ctx.lib.pbq_p2p_sum(ctx.handle, ptr(slots), int(slot), int(world), int(n), ptr(out), ptr(cnt),
                                 ctypes.c_uint32(target), ptr(status), stream_ptr(out.device))
        ctx.check(st, "p2p_sum")


def p2p_wait(ctx, cnt, target, status):
    with ctx.lock:
        st = ctx.lib.pbq_p2p_wait(ctx.handle, ptr(cnt), ctypes.c_uint32(target), ptr(status), stream_ptr(cnt.device))
        ctx.check(st, "p2p_wait")


def xchg_expected_tiles(ctx, n2, n, S, rank, world):
    t = ctypes.c_uint32()
    ctx.check(ctx.lib.pbq_xchg_expected_tiles(n2, n, S, rank, world, ctypes.byref(t)), "xchg_expected_tiles")
    return int(t.value)


def householder_qr_(ctx, a, r=None, want_q=True, rank_flag=None):
    """In-place QR of the m×n device matrix ``a`` (must be kernel-ready)."""
    dev = a.device
    m, n = a.shape
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_qr_workspace_bytes(ctx.handle, m, n, ctypes.byref(nbytes)), "qr workspace")
        ws = workspace(nbytes.value, dev)
        st = ctx.lib.pbq_householder_qr(ctx.handle, m, n, ptr(a), ld_of(a), ptr(r), ld_of(r) if r is not None else 0,
                                        int(bool(want_q)), ptr(rank_flag), ptr(ws), nbytes.value, stream_ptr(dev))
        ctx.check(st, "householder_qr")
    return a, r


def orth_basis_(ctx, a, out=None, rank_flag=None):
    """Basis-only orth of the m×n device matrix ``a`` (kernel-ready; clobbered):
    returns B = Q·T (T upper triangular, positive diagonal, near the identity)
    for an operand that is multiplied and orthonormalised again
    (``pbq_orth_basis``; the intermediate orth calls of algorithms.py:196-205)."""
    dev = a.device
    m, n = a.shape
    if out is None:
        out = empty_matrix(m, n, dev)
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_qr_workspace_bytes(ctx.handle, m, n, ctypes.byref(nbytes)), "qr workspace")
        ws = workspace(nbytes.value, dev)
        st = ctx.lib.pbq_orth_basis(ctx.handle, m, n, ptr(a), ld_of(a), ptr(out), ld_of(out), ptr(rank_flag), ptr(ws),
                                    nbytes.value, stream_ptr(dev))
        ctx.check(st, "orth_basis")
    return out


def residual_fro(ctx, a, q, l, p, out=None):
    """out[0] = ‖a − q·l·pᵀ‖_F², out[1] = ‖a‖_F² (device float64[2]), in one
    pass over ``a`` (q: n1×k, l: k×k, p: n2×k)."""
    dev = a.device
    a, q, l, p = (as_kernel_operand(t) for t in (a, q, l, p))
    n1, n2 = a.shape
    k = l.shape[0]
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=dev)
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_residual_workspace_bytes(ctx.handle, n1, n2, k, ctypes.byref(nbytes)), "residual workspace")
        ws = workspace(nbytes.value, dev)
        st = ctx.lib.pbq_residual_fro(ctx.handle, n1, n2, k, ptr(a), ld_of(a), ptr(q), ld_of(q), ptr(l), ld_of(l),
                                      ptr(p), ld_of(p), ptr(out), ptr(ws), nbytes.value, stream_ptr(dev))
        ctx.check(st, "residual_fro")
    return out


def gaussian(ctx, rows, cols, seed, device, row_offset=0, out=None, status=None):
    """Enqueue the sketch; ``status`` (int32 device tensor) receives the
    generator's overflow flag (callers check it when they synchronise)."""
    if out is None:
        out = empty_matrix(rows, cols, device)
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_gaussian_workspace_bytes(ctx.handle, rows, cols, row_offset, ctypes.byref(nbytes)),
                  "gaussian workspace")
        ws = workspace(nbytes.value, device)
        st = ctx.lib.pbq_gaussian(ctx.handle, rows, cols, row_offset, seed & ((1 << 64) - 1), seed >> 64, ptr(out),
                                  ld_of(out), ptr(status), ptr(ws), nbytes.value, stream_ptr(device))
        ctx.check(st, "gaussian")
    return out


def transpose(ctx, src, dst=None, lower=False):
    n = src.shape[0]
    if dst is None:
        dst = empty_matrix(n, n, src.device)
    with ctx.lock:
        st = ctx.lib.pbq_transpose(ctx.handle, n, ptr(src), ld_of(src), ptr(dst), ld_of(dst), int(bool(lower)),
                                   stream_ptr(src.device))
        ctx.check(st, "transpose")
    return dst


def second_stage(ctx, r, w=None, l=None):
    """(W, R̃) = qr(Rᵀ) and L = tril(R̃ᵀ) of the d×d upper-triangular ``r``
    (reference algorithms.py:256-257) → (W, L)."""
    d = r.shape[0]
    dev = r.device
    w = empty_matrix(d, d, dev) if w is None else w
    l = empty_matrix(d, d, dev) if l is None else l
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_second_stage_workspace_bytes(ctx.handle, d, ctypes.byref(nbytes)), "second stage workspace")
        ws = workspace(nbytes.value, dev)
        st = ctx.lib.pbq_second_stage(ctx.handle, d, ptr(r), ld_of(r), ptr(w), ld_of(w), ptr(l), ld_of(l), ptr(ws),
                                      nbytes.value, stream_ptr(dev))
        ctx.check(st, "second stage")
    return w, l


def jacobi_svd(ctx, x, accumulate=True, want_y=True, status=None, precondition=True):
    """One-sided Jacobi SVD of the rows of ``x`` (n×L, n ≤ L):
    G·x = diag(s)·Y (pbq_jacobi_svd).  ``precondition`` first reduces x to
    the n×n R̃ of xᵀ = Q·R, Rᵀ = W·R̃ (LAPACK dgejsv's QR preconditioning;
    leave it off when x already is such a factor).  Returns (s, Y, G, status)
    as device tensors — Y None unless ``want_y``, G None unless
    ``accumulate``; status = [sweeps, not-converged flag] (int32, on the
    device)."""
    x = as_kernel_operand(x)
    n, L = x.shape
    dev = x.device
    s = torch.empty(n, dtype=torch.float64, device=dev)
    y = empty_matrix(n, L, dev) if want_y else None
    g = empty_matrix(n, n, dev) if accumulate else None
    if status is None:
        status = torch.zeros(2, dtype=torch.int32, device=dev)
    flags = (JACOBI_ACCUMULATE if accumulate else 0) | (JACOBI_PRECONDITION if precondition else 0)
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_jacobi_svd_workspace_bytes(ctx.handle, n, L, flags, ctypes.byref(nbytes)),
                  "jacobi_svd workspace")
        ws = workspace(nbytes.value, dev)
        st = ctx.lib.pbq_jacobi_svd(ctx.handle, n, L, ptr(x), ld_of(x), flags, ptr(s), ptr(y),
                                    ld_of(y) if y is not None else 0, ptr(g), ld_of(g) if g is not None else 0,
                                    ptr(status), ptr(ws), nbytes.value, stream_ptr(dev))
        ctx.check(st, "jacobi_svd")
    return s, y, g, status


def cpqr_pivots(ctx, m, out=None):
    """Pivot order of LAPACK dgeqp3 for the m×n device matrix ``m`` → int64
    device tensor ``perm`` (n entries) with m[:, perm] = Q·R."""
    dev = m.device
    m = as_kernel_operand(m)
    rows, cols = m.shape
    if out is None:
        out = torch.empty(cols, dtype=torch.int64, device=dev)
    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_cpqr_workspace_bytes(ctx.handle, rows, cols, ctypes.byref(nbytes)), "cpqr workspace")
        ws = workspace(nbytes.value, dev)
        st = ctx.lib.pbq_cpqr_pivots(ctx.handle, rows, cols, ptr(m), ld_of(m), ptr(out), ptr(ws), nbytes.value,
                                     stream_ptr(dev))
        ctx.check(st, "cpqr_pivots")
    return out


def gather_columns(ctx, src, perm, out=None):
    """out[:, i] = src[:, perm[i]] (perm: int64 device tensor)."""
    src = as_kernel_operand(src)
    rows, cols = src.shape[0], perm.shape[0]
    if out is None:
        out = empty_matrix(rows, cols, src.device)
    with ctx.lock:
        st = ctx.lib.pbq_gather_columns(ctx.handle, rows, cols, ptr(src), ld_of(src), ptr(perm), ptr(out),
                                        ld_of(out), stream_ptr(src.device))
        ctx.check(st, "gather_columns")
    return out
