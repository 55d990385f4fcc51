"""TEST INFRASTRUCTURE: a CPU backend for DistributedPbpQlp built from the
oracle (numpy/LAPACK + the C sketch restatement), so the row-sharded
orchestration and its collectives run under `gloo` without a GPU."""
import numpy as np
import torch

from oracle.pbp_qlp_oracle import c_gaussian, oracle_qr, rank_flag


class NumpyBackend:
    device = torch.device("cpu")

    def empty(self, rows, cols):
        return torch.empty((rows, cols), dtype=torch.float64)

    def zeros_i32(self, n):
        return torch.zeros(n, dtype=torch.int32)

    def gaussian(self, rows, cols, seed, row_offset, status=None):
        return torch.from_numpy(c_gaussian(rows, cols, seed, row_offset=row_offset))

    def gemm_tn(self, a, x, out, nonfinite=None):
        if nonfinite is not None and not torch.isfinite(a).all():
            nonfinite.fill_(1)
        out.copy_(torch.from_numpy(a.numpy().T @ x.numpy()))
        return out

    def gemm_nn(self, a, x, out):
        out.copy_(torch.from_numpy(a.numpy() @ x.numpy()))
        return out

    def qr_(self, m, r, flag=None):
        q, rr = oracle_qr(m.numpy())
        m.copy_(torch.from_numpy(q))
        r.copy_(torch.from_numpy(rr))
        if flag is not None:
            flag.fill_(rank_flag(rr))

    def transpose(self, src, dst, lower=False):
        t = src.T
        dst.copy_(torch.tril(t) if lower else t)
        return dst

    def contiguous(self, t):
        return t.contiguous()
