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

    # -- distributed Cholesky-QR2, restated for the CPU (pbq_cholqr2_dist) --
    KAPPA_MAX = 1e6  # the device guard (pbq_api.cu CQ_KAPPA_MAX)
    KAPPA_MAX_BASIS = 3e7  # … of the basis-only stage 3 (CQ_KAPPA_MAX_BASIS)

    def cholqr2_dist_state(self, m, n):
        return {"G": torch.zeros((n, n), dtype=torch.float64), "fallback": torch.zeros(1, dtype=torch.int32)}

    def cholqr2_dist(self, stage, a, r, state, flag=None):
        import scipy.linalg as sla

        g = state["G"]
        if stage == 0:
            state["fallback"].zero_()
            g.copy_(torch.from_numpy(a.numpy().T @ a.numpy()))
            return
        if state["fallback"].item():
            return
        if stage in (1, 3):
            try:
                r1 = np.linalg.cholesky(g.numpy()).T
            except np.linalg.LinAlgError:
                state["fallback"].fill_(1)
                return
            r1i = sla.solve_triangular(r1, np.eye(r1.shape[0]), lower=False)
            if not np.linalg.norm(r1, 1) * np.linalg.norm(r1i, 1) <= (self.KAPPA_MAX_BASIS if stage == 3 else self.KAPPA_MAX):
                state["fallback"].fill_(1)
                return
            q1 = a.numpy() @ r1i
            if stage == 3:  # basis-only finish: a ← A·R₁⁻¹ = Q·R₂
                a.copy_(torch.from_numpy(q1))
                if flag is not None:
                    flag.fill_(0)
                return
            state["r1"], state["q1"] = r1, q1
            g.copy_(torch.from_numpy(q1.T @ q1))
            return
        try:
            r2 = np.linalg.cholesky(g.numpy()).T
        except np.linalg.LinAlgError:
            state["fallback"].fill_(1)
            return
        rr = r2 @ state["r1"]
        r.copy_(torch.from_numpy(np.triu(rr)))
        a.copy_(torch.from_numpy(sla.solve_triangular(r2, state["q1"].T, trans="T", lower=False).T))
        if flag is not None:
            flag.fill_(rank_flag(rr))


class FakeP2PBackend(NumpyBackend):
    """NumpyBackend plus a stand-in for the peer-memory exchange
    (CudaBackend.xchg_init / xchg_at_x / p2p_allreduce / p2p_allgather_rows),
    its data movement done with gloo collectives.  ``fault`` injects the
    failures the exchange's init self-check must catch:
      None       a working transport;
      "wrong"    rank 1's AᵀX result is corrupted (a broken peer mapping);
      "timeout"  rank 0's status word reports a spin timeout."""

    def __init__(self, fault=None):
        self.fault = fault

    def xchg_init(self, n2, d, group):
        import torch.distributed as dist

        from paper_2103_07245_b200.distributed import _XchgBuffers, _gram_np, xchg_slice_rows

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        S, ldl = xchg_slice_rows(n2, world), d + (d & 1)
        land = torch.zeros(world * S * ldl, dtype=torch.float64)
        c = torch.zeros(world * S * ldl, dtype=torch.float64)
        ctr = torch.zeros(64, dtype=torch.int32)
        gram = torch.zeros(2 * world * _gram_np(d) ** 2, dtype=torch.float64)
        x = _XchgBuffers(rank, world, S, ldl, land, c, ctr, gram)
        x.group = group
        return x

    def xchg_at_x(self, xchg, a, x, n2, epoch, nonfinite=None):
        import torch.distributed as dist

        d = x.shape[1]
        part = torch.from_numpy(a.numpy().T @ x.numpy())
        if nonfinite is not None and not torch.isfinite(a).all():
            nonfinite.fill_(1)
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=xchg.group)
        if self.fault == "wrong" and xchg.rank == 1:
            part[0, 0] += 1.0
        if self.fault == "timeout" and xchg.rank == 0:
            xchg.status.fill_(1)
        xchg.C[:n2, :d].copy_(part)

    def p2p_allreduce(self, xchg, g, epoch):
        import torch.distributed as dist

        dist.all_reduce(g, op=dist.ReduceOp.SUM, group=xchg.group)

    def p2p_allgather_rows(self, xchg, epoch):
        import torch.distributed as dist

        S = xchg.S
        mine = xchg.C[xchg.rank * S:(xchg.rank + 1) * S].contiguous()
        parts = [torch.empty_like(mine) for _ in range(xchg.world)]
        dist.all_gather(parts, mine, group=xchg.group)
        xchg.C.copy_(torch.cat(parts, 0))
