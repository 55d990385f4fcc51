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
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np
import torch

from . import _lib
from . import device as _dev
from . import exceptions as _exc
from .linalg import HostMatrix, from_device, householder_qr, to_device_matrix, warn_rank
from .validation import check_index_range, check_seed, check_sketch_params

__all__ = ["SketchRecord", "QlpFactors", "pbp_qlp", "pbp_qlp_flops", "pbp_qlp_bytes"]


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


def pbp_qlp(a, d, q=0, seed=0, reorthonormalize=True, *, phi=None, device=None):
    """Projection-based partial QLP factorization of ``a`` on the GPU.

    Same signature, arguments, errors, warnings and return fields as the
    reference (algorithms.py:209-260).  Extensions (keyword-only):
    ``phi`` supplies the sketch explicitly (oracle mode, n1×d); ``device``
    picks the GPU for array-like inputs.  numpy/array-like input returns numpy
    factors; a torch tensor returns torch tensors on the tensor's device.
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
    seed = check_seed(seed)
    kind, home = ha.kind, ha.home
    A = ha.to_device(device)
    dev = A.device
    ctx = _dev.context(dev)

    Q = _dev.empty_matrix(n1, d, dev)
    P = _dev.empty_matrix(n2, d, dev)
    L = _dev.empty_matrix(d, d, dev)
    R = _dev.empty_matrix(d, d, dev)
    flags = torch.zeros(2 * q + 2, dtype=torch.int32, device=dev)  # [status, rank flags...]
    prob = _lib.PbqProblem()
    prob.n1, prob.n2, prob.d, prob.q = n1, n2, d, q
    prob.a, prob.lda = A.data_ptr(), A.stride(0)
    prob.seed_lo, prob.seed_hi = seed & ((1 << 64) - 1), seed >> 64
    prob.reorthonormalize = 1 if reorthonormalize else 0
    prob.check_finite = 1
    out = _lib.PbqOutputs()
    out.q, out.ldq = Q.data_ptr(), Q.stride(0)
    out.l, out.ldl = L.data_ptr(), L.stride(0)
    out.p, out.ldp = P.data_ptr(), P.stride(0)
    out.r, out.ldr = R.data_ptr(), R.stride(0)
    if phi is not None:
        pkind, PHI, _, _ = to_device_matrix(phi, "phi", dev)
        if tuple(PHI.shape) != (n1, d):
            raise _exc.DimensionError(f"phi must have shape ({n1}, {d}), got {tuple(PHI.shape)}")
        prob.phi, prob.ldphi = PHI.data_ptr(), PHI.stride(0)
        sketch_phi = phi if kind == "torch" or isinstance(phi, np.ndarray) else np.asarray(phi, dtype=np.float64)
    else:
        PHI = _dev.empty_matrix(n1, d, dev)
        prob.phi, prob.ldphi = None, 0
        out.phi, out.ldphi = PHI.data_ptr(), PHI.stride(0)
        sketch_phi = None
    out.nonfinite = flags.data_ptr()
    out.rank_flags = flags.data_ptr() + 4

    nbytes = ctypes.c_size_t()
    with ctx.lock:
        ctx.check(ctx.lib.pbq_pbp_qlp_workspace_bytes(ctx.handle, ctypes.byref(prob), ctypes.byref(nbytes)),
                  "pbp_qlp workspace")
        ws = _dev.workspace(nbytes.value, dev)
        st = ctx.lib.pbq_pbp_qlp(ctx.handle, ctypes.byref(prob), ctypes.byref(out), _dev.ptr(ws), nbytes.value,
                                 _dev.stream_ptr(dev))
        ctx.check(st, "pbp_qlp")
    fl = flags.cpu().tolist()  # the one device→host synchronisation
    if fl[0] & 1:
        raise _exc.MatrixInputError("a contains non-finite entries")
    if fl[0] & 2:
        raise _exc.DeviceError("sketch generator overflow (internal error)")
    for flag in fl[1:]:
        warn_rank(flag, stacklevel=3)

    passes = 2 * q + 2
    if sketch_phi is not None:
        sketch = SketchRecord(PHI, kind, seed, d, q, passes, home)
        if kind == "numpy":
            sketch._host = np.asarray(sketch_phi, dtype=np.float64)
    else:
        sketch = SketchRecord(PHI, kind, seed, d, q, passes, home)
    return QlpFactors(
        from_device(Q, kind, home),
        from_device(L, kind, home),
        from_device(P, kind, home),
        from_device(R, kind, home),
        sketch,
    )
