"""Dense kernels of the PbP-QLP path, on the GPU.

Drop-in counterparts of the reference's ``gaussian_matrix``,
``householder_qr`` and ``orth`` (/root/reference/pkg/src/pbpqlp/linalg.py:83-165).
Inputs may be numpy arrays / array-likes (results come back as numpy) or
torch tensors (results stay torch, on the input's device).  All arithmetic runs
in libpbq's sm_100a kernels.
"""
import warnings
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import device as _dev
from . import exceptions as _exc
from .validation import check_count, check_seed, coerce_host_matrix, check_shape

__all__ = ["QrFactors", "gaussian_matrix", "householder_qr", "column_pivoted_qr", "orth", "RANK_DEFICIENCY_RTOL"]

#: Columns whose pivot falls below this multiple of the leading pivot are
#: reported as numerically dependent by :func:`orth` (linalg.py:48).
RANK_DEFICIENCY_RTOL = 1e-14

_RANK_MSG = {
    1: "orth: input is numerically rank deficient; trailing basis directions are arbitrary",
    2: "orth: input is identically zero; returned basis is arbitrary",
}


class QrFactors(NamedTuple):
    """Economy-size QR factors (linalg.py:51-60): ``q`` orthonormal columns,
    ``r`` upper triangular with nonnegative diagonal."""

    q: object
    r: object
    perm: Optional[object] = None


def warn_rank(flag, stacklevel=3):
    """Re-emit the reference's orth warning (linalg.py:152-164) for a device flag."""
    msg = _RANK_MSG.get(int(flag))
    if msg:
        warnings.warn(msg, _exc.RankDeficiencyWarning, stacklevel=stacklevel)


class HostMatrix:
    """A validated matrix argument before it touches the device.

    ``kind`` is "numpy" for array-likes (results returned as numpy) and
    "torch" for tensors (results returned as tensors on ``home``).
    """

    def __init__(self, m, name):
        if isinstance(m, torch.Tensor):
            check_shape(m.shape, m.dim(), name)
            if m.is_complex():
                raise _exc.MatrixInputError(f"{name} is not numeric: complex input")
            self.kind, self.tensor, self.array, self.home = "torch", m.detach(), None, m.device
        else:
            self.kind, self.tensor, self.array, self.home = "numpy", None, coerce_host_matrix(m, name), None
        self.shape = tuple(self.tensor.shape if self.tensor is not None else self.array.shape)

    def host_tensor(self):
        """CPU float64 contiguous torch view/copy of a host input, else None."""
        if self.array is not None:
            return torch.from_numpy(np.ascontiguousarray(self.array))
        t = self.tensor
        if t.is_cuda:
            return None
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        return t.contiguous()

    def all_finite(self):
        if self.array is not None:
            return bool(np.isfinite(self.array).all())
        return bool(torch.isfinite(self.tensor).all().item())

    def to_device(self, device=None):
        """Kernel-ready float64 CUDA copy/view (row-major, even row stride)."""
        if self.tensor is not None:
            t = self.tensor
            dev = _dev.require_cuda(t.device if t.is_cuda else device)
            if t.dtype != torch.float64:
                t = t.to(torch.float64)
            if not t.is_cuda:
                out = _dev.empty_matrix(t.shape[0], t.shape[1], dev)
                return _dev.h2d(t.contiguous(), out)
            return _dev.as_kernel_operand(t)
        dev = _dev.require_cuda(device)
        arr = self.array
        out = _dev.empty_matrix(arr.shape[0], arr.shape[1], dev)
        return _dev.h2d(torch.from_numpy(np.ascontiguousarray(arr)), out)


def to_device_matrix(m, name, device=None):
    """(kind, device tensor, host numpy or None, home device) for ``m``."""
    h = m if isinstance(m, HostMatrix) else HostMatrix(m, name)
    return h.kind, h.to_device(device), h.array, h.home


# device → numpy results of at least this size travel through a pinned host
# buffer (one DMA at link speed; the runtime's pageable path moves a 41 MB
# factor in 19 ms, ~2 GB/s, against 1 ms)
PINNED_D2H_MIN_BYTES = 1 << 20


def from_device(t, kind, home=None):
    """Return a device result in the caller's array type."""
    if kind == "numpy":
        if t.is_cuda and t.numel() * t.element_size() >= PINNED_D2H_MIN_BYTES:
            try:
                buf = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
            except RuntimeError:  # no pinned memory left: the pageable path
                buf = None
            if buf is not None:
                buf.copy_(t, non_blocking=True)
                torch.cuda.current_stream(t.device).synchronize()
                return buf.numpy()
        return t.cpu().numpy() if t.is_contiguous() else t.contiguous().cpu().numpy()
    t = t.contiguous()
    if home is not None and torch.device(home) != t.device:
        return t.to(home)
    return t


def gaussian_matrix(rows, cols, seed=0, *, device=None, as_tensor=False, row_offset=0):
    """``rows × cols`` standard normals, bitwise equal to the reference's
    ``gaussian_matrix`` (linalg.py:83-93: numpy Philox(key=seed) +
    ``standard_normal``), generated on the GPU.

    ``row_offset`` returns rows ``[row_offset, row_offset + rows)`` of the
    same stream layout (used by the row-sharded multi-GPU path).
    """
    rows = check_count(rows, "rows")
    cols = check_count(cols, "cols")
    seed = check_seed(seed)
    dev = _dev.require_cuda(device)
    ctx = _dev.context(dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    out = _dev.gaussian(ctx, rows, cols, seed, dev, row_offset=int(row_offset), status=status)
    if int(status.item()):
        raise _exc.DeviceError("sketch generator overflow (internal error)")
    return out if as_tensor else from_device(out, "numpy")


def _qr(m, want_flag):
    kind, t, _host, home = to_device_matrix(m, "m")
    dev = t.device
    ctx = _dev.context(dev)
    n1, n2 = t.shape
    if n1 < n2:
        raise _exc.DeviceError("householder_qr on the GPU supports m >= n (tall or square) matrices")
    if t is m or (isinstance(m, torch.Tensor) and t.data_ptr() == m.data_ptr()):
        t = _dev.as_kernel_operand(t.clone())
    if not torch.isfinite(t).all().item():
        raise _exc.MatrixInputError("m contains non-finite entries")
    r = _dev.empty_matrix(n2, n2, dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev) if want_flag else None
    _dev.householder_qr_(ctx, t, r, want_q=True, rank_flag=flag)
    out = QrFactors(from_device(t, kind, home), from_device(r, kind, home), None)
    return out, (int(flag.item()) if want_flag else 0)


def householder_qr(m):
    """Unpivoted Householder QR with economy factors and ``diag(r) >= 0``
    (linalg.py:106-115)."""
    return _qr(m, False)[0]


def orth(m):
    """Orthonormal basis for the range of ``m`` (linalg.py:142-165); warns with
    :class:`RankDeficiencyWarning` exactly when the reference does."""
    f, flag = _qr(m, True)
    warn_rank(flag, stacklevel=3)
    return f.q


def cpqr_device(ctx, t):
    """Column-pivoted QR of the m×n device matrix ``t`` → (q, r, perm) device
    tensors: perm from the dgeqp3-rule pivot kernel, then the unpivoted QR of
    the gathered columns (identical reflector sequence).  Economy sizes as
    scipy: q m×k, r k×n, k = min(m, n)."""
    m, n = t.shape
    dev = t.device
    perm = _dev.cpqr_pivots(ctx, t)
    g = _dev.gather_columns(ctx, t, perm)
    k = min(m, n)
    if m >= n:
        r = _dev.empty_matrix(n, n, dev)
        _dev.householder_qr_(ctx, g, r, want_q=True)
        return g, r, perm
    q = _dev.as_kernel_operand(g[:, :m].clone())
    r11 = _dev.empty_matrix(k, k, dev)
    _dev.householder_qr_(ctx, q, r11, want_q=True)
    r = _dev.empty_matrix(k, n, dev)
    r[:, :k] = r11
    r[:, k:] = _dev.gemm(ctx, q, _dev.as_kernel_operand(g[:, k:]), trans_a=True)  # R12 = Qᵀ·M[:, perm[k:]]
    return q, r, perm


def column_pivoted_qr(m):
    """Column-pivoted Householder QR with nonincreasing pivot magnitudes
    (linalg.py:118-129): ``m[:, perm] = q @ r``, ``diag(r) >= 0``, pivots as
    LAPACK dgeqp3 chooses them (exact ties → the lowest current position)."""
    kind, t, _host, home = to_device_matrix(m, "m")
    if not torch.isfinite(t).all().item():
        raise _exc.MatrixInputError("m contains non-finite entries")
    ctx = _dev.context(t.device)
    q, r, perm = cpqr_device(ctx, t)
    r = torch.triu(r)
    if kind == "numpy":
        return QrFactors(from_device(q, kind), from_device(r, kind), perm.cpu().numpy().astype(np.int32))
    return QrFactors(from_device(q, kind, home), from_device(r, kind, home), perm.to(home))
