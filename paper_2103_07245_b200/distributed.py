"""Row-sharded multi-GPU PbP-QLP.

Rank g of G owns the contiguous row block A_g = A[r_g : r_{g+1}] and the
matching rows Φ_g of the sketch (the device generator produces any row range
of the global stream, so Φ does not depend on G).  Exchanges:

* AᵀX = Σ_g A_gᵀ X_g — the local GEMM runs in ``chunks`` column blocks of
  A_g (row blocks of the n2×d result) and each block's NCCL allreduce(sum)
  is issued asynchronously right after its GEMM is enqueued: the collective
  is ordered after the work already on the stream, so the exchange of block
  b overlaps the GEMM of block b+1 and only the last block's allreduce is
  exposed.  The result is identical on all ranks, so ``orth`` of it is
  computed replicated (same input → same bits).
* qr(A·P̄) — A_g·P̄ is local; its QR is a distributed Cholesky-QR2
  (``pbq_cholqr2_dist``): local Gram A_gᵀA_g, allreduce(sum) of the d×d Gram,
  the guarded factorization replicated (same G → same R on every rank), the
  local product, and again for the second pass — two d×d allreduces and no
  tall replicated work.  Its fallback is the TSQR tree: local QR (Q_g, R_g),
  all-gather of the d×d R factors, a replicated QR of the stacked (G·d)×d
  matrix → (Q̂, R), then Q_g ← Q_g·Q̂_g (local GEMM).
* No host synchronisation inside ``run``: each distributed Cholesky-QR2 ORs
  its κ-guard flag into a device flag (identical on every rank, since every
  rank factors the same allreduced Gram).  ``finish`` reads it with the
  status flags in its one device→host copy; when a guard fired, every rank
  re-runs the factorization with the fallbacks (TSQR, replicated orth) in
  every QR.  Well-conditioned inputs therefore never stall the stream.
* qr(Rᵀ), L = tril(R̃ᵀ) and P = P̄·W are replicated.

Q stays row-sharded (rank g holds Q[r_g : r_{g+1}]); L, P, R are replicated.
The local arithmetic goes through a backend: :class:`CudaBackend` (libpbq's
sm_100a kernels through the C ABI) in the product.  The CPU ``gloo`` tests
substitute a numpy backend defined in tests/ to exercise exactly this
orchestration without a GPU.
"""
import ctypes

import torch
import torch.distributed as dist

from . import device as _dev
from . import exceptions as _exc
from .linalg import warn_rank

__all__ = ["shard_rows", "DistributedPbpQlp", "CudaBackend", "P2PExchange", "virtual_exchanges",
           "xchg_slice_rows"]


def shard_rows(n1, world):
    """Contiguous, balanced row offsets [r_0 = 0, …, r_G = n1]."""
    return [(n1 * g) // world for g in range(world + 1)]


# ------------------------------------------------ fused AᵀX exchange (p2p) --
def xchg_slice_rows(n2, world):
    """Rows per owner slice of the exchanged n2×d result: ⌈n2/G⌉ rounded up
    to the GEMM's 128-row tile, so no tile straddles two owners."""
    s = -(-n2 // world)
    return -(-s // 128) * 128


class _XchgBuffers:
    """One rank's landing buffer (G slots of S×ldl), result C (G·S×ldl), tile
    and done counters, and device arrays of every rank's pointers to them
    (indexed by rank) — the arguments of pbq_gemm_tn_scatter /
    pbq_xchg_reduce / pbq_xchg_wait (include/pbq.h)."""

    def __init__(self, rank, world, S, ldl, land, c, ctr, gram):
        self.rank, self.world, self.S, self.ldl = rank, world, S, ldl
        self.land = land.view(world * S, ldl)
        self.C = c.view(world * S, ldl)
        # counter block [AᵀX tiles, AᵀX done, status, Gram pushes, all-gather pushes]
        self.cnt, self.done, self.status = ctr[0:1], ctr[1:2], ctr[2:3]
        self.gram_cnt, self.ag_cnt = ctr[3:4], ctr[4:5]
        # Gram allreduce landing: two halves (epoch parity) of `world` slots of
        # np² doubles — a fast peer's next push lands in the other half
        self.gram_land = gram
        self.gram_slot = gram.numel() // (2 * world)
        self.land_ptrs = self.c_ptrs = self.cnt_ptrs = self.done_ptrs = None

    def set_peers(self, land, c, ctr, gram):
        dev = self.land.device
        mk = lambda v: torch.tensor([int(x) for x in v], dtype=torch.int64, device=dev)  # noqa: E731
        self.land_ptrs, self.c_ptrs = mk(land), mk(c)
        self.cnt_ptrs, self.done_ptrs = mk(ctr), mk([x + 4 for x in ctr])
        self.gram_cnt_ptrs, self.ag_cnt_ptrs = mk([x + 12 for x in ctr]), mk([x + 16 for x in ctr])
        half = self.gram_slot * self.world * 8
        self.gram_ptrs = (mk(gram), mk([x + half for x in gram]))


def _gram_np(d):
    return 32 * (-(-d // 32))


class P2PExchange(_XchgBuffers):
    """The buffers in symmetric memory (torch.distributed._symmetric_memory:
    peer-mapped allocations over NVLink) of this rank of ``group``."""

    def __init__(self, n2, d, device, group=None):
        import torch.distributed._symmetric_memory as symm

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        S, ldl = xchg_slice_rows(n2, world), d + (d & 1)
        pg = group if group is not None else dist.group.WORLD
        land = symm.empty(world * S * ldl, dtype=torch.float64, device=device)
        c = symm.empty(world * S * ldl, dtype=torch.float64, device=device)
        ctr = symm.empty(64, dtype=torch.int32, device=device)
        gram = symm.empty(2 * world * _gram_np(d) ** 2, dtype=torch.float64, device=device)
        c.zero_()  # rows ≥ n2 of C stay zero (orth(C) runs on whole row slices)
        ctr.zero_()
        super().__init__(rank, world, S, ldl, land, c, ctr, gram)
        bufs = (land, c, ctr, gram)
        handles = [symm.rendezvous(t, pg) for t in bufs]
        peers = []
        for t, h in zip(bufs, handles):
            off = t.data_ptr() - int(h.buffer_ptrs[rank])
            peers.append([int(h.buffer_ptrs[p]) + off for p in range(world)])
        self.set_peers(*peers)
        self._keep = (bufs, handles)
        torch.cuda.synchronize(device)
        dist.barrier(group)  # every rank's counters are zero before any peer adds to them


def virtual_exchanges(n2, d, world, device):
    """``world`` exchange buffer sets on ONE device whose peer pointers refer
    to each other — the one-GPU emulation of the p2p exchange used by the
    tests (each virtual rank's kernels are launched in turn; no kernel waits
    on a kernel that has not run yet)."""
    S, ldl = xchg_slice_rows(n2, world), d + (d & 1)
    xs = []
    for r in range(world):
        land = torch.full((world * S * ldl,), float("nan"), dtype=torch.float64, device=device)
        c = torch.zeros(world * S * ldl, dtype=torch.float64, device=device)
        ctr = torch.zeros(64, dtype=torch.int32, device=device)
        gram = torch.full((2 * world * _gram_np(d) ** 2,), float("nan"), dtype=torch.float64, device=device)
        xs.append(_XchgBuffers(r, world, S, ldl, land, c, ctr, gram))
    for x in xs:
        x.set_peers([y.land.data_ptr() for y in xs], [y.C.data_ptr() for y in xs], [y.cnt.data_ptr() for y in xs],
                    [y.gram_land.data_ptr() for y in xs])
    return xs


class CudaBackend:
    """Local kernels of one rank: libpbq through the C ABI (no CPU path)."""

    def __init__(self, device):
        self.device = _dev.require_cuda(device)
        self.ctx = _dev.context(self.device)

    def empty(self, rows, cols):
        return _dev.empty_matrix(rows, cols, self.device)

    def zeros_i32(self, n):
        return torch.zeros(n, dtype=torch.int32, device=self.device)

    def gaussian(self, rows, cols, seed, row_offset, status=None):
        return _dev.gaussian(self.ctx, rows, cols, seed, self.device, row_offset=row_offset, status=status)

    def gemm_tn(self, a, x, out, nonfinite=None):
        return _dev.gemm(self.ctx, a, x, trans_a=True, out=out, nonfinite=nonfinite)

    def gemm_nn(self, a, x, out):
        return _dev.gemm(self.ctx, a, x, trans_a=False, out=out)

    def qr_(self, m, r, flag=None):
        """In-place thin QR of m (m ≥ n); R into r; rank test into flag[0]."""
        _dev.householder_qr_(self.ctx, m, r, want_q=True, rank_flag=flag)

    def transpose(self, src, dst, lower=False):
        return _dev.transpose(self.ctx, src, dst, lower=lower)

    # -- fused AᵀX exchange over peer memory ----------------------------------
    def xchg_init(self, n2, d, group):
        return P2PExchange(n2, d, self.device, group)

    def p2p_allreduce(self, xchg, g, epoch):
        """g (the np×np Gram) ← Σ over ranks, by pushes into every rank's slot
        and a slot-ordered sum (call ``epoch`` ≥ 1 of this buffer set)."""
        self.p2p_allreduce_push(xchg, g, epoch)
        self.p2p_allreduce_sum(xchg, g, epoch)

    def p2p_allreduce_push(self, xchg, g, epoch):
        n = g.numel()
        if n > xchg.gram_slot:
            raise _exc.ParameterError("p2p allreduce: buffer larger than the Gram slot")
        _dev.p2p_push(self.ctx, g, n, xchg.gram_ptrs[epoch & 1], xchg.gram_slot, xchg.rank, xchg.world,
                      xchg.gram_cnt_ptrs)

    def p2p_allreduce_sum(self, xchg, g, epoch):
        slots = xchg.gram_land[(epoch & 1) * xchg.world * xchg.gram_slot:]
        _dev.p2p_sum(self.ctx, slots, xchg.gram_slot, xchg.world, g.numel(), g, xchg.gram_cnt,
                     epoch * 64 * xchg.world, xchg.status)

    def p2p_allgather_rows(self, xchg, epoch):
        """Every rank's S-row slice of xchg.C into every rank's C."""
        self.p2p_allgather_push(xchg)
        self.p2p_allgather_wait(xchg, epoch)

    def p2p_allgather_push(self, xchg):
        slot = xchg.S * xchg.ldl
        mine = xchg.C[xchg.rank * xchg.S:(xchg.rank + 1) * xchg.S]
        _dev.p2p_push(self.ctx, mine, slot, xchg.c_ptrs, slot, xchg.rank, xchg.world, xchg.ag_cnt_ptrs)

    def p2p_allgather_wait(self, xchg, epoch):
        _dev.p2p_wait(self.ctx, xchg.ag_cnt, epoch * 64 * xchg.world, xchg.status)

    def xchg_at_x(self, xchg, a, x, n2, epoch, nonfinite=None):
        """xchg.C[:n2] = Σ_g A_gᵀ·X_g on every rank: scatter GEMM, slice
        reduce + all-gather, wait (call ``epoch`` ≥ 1 of this buffer set)."""
        d = x.shape[1]
        _dev.gemm_tn_scatter(self.ctx, a, x, xchg, nonfinite=nonfinite)
        tiles = _dev.xchg_expected_tiles(self.ctx, n2, d, xchg.S, xchg.rank, xchg.world)
        _dev.xchg_reduce(self.ctx, xchg, n2, d, epoch * tiles)
        _dev.xchg_wait(self.ctx, xchg, epoch * 64 * xchg.world)

    def second_stage(self, r, w, l):
        """(W, R̃) = qr(Rᵀ), L = tril(R̃ᵀ) (one CTA for d ≤ 160)."""
        return _dev.second_stage(self.ctx, r, w, l)

    def contiguous(self, t):
        return _dev.as_kernel_operand(t)

    # -- distributed Cholesky-QR2 (pbq_cholqr2_dist) -------------------------
    def cholqr2_dist_state(self, m, n):
        """Persistent (workspace, G, fallback flag) for one m×n shard shape."""
        nbytes, ldg = ctypes.c_size_t(), ctypes.c_int64()
        self.ctx.check(self.ctx.lib.pbq_cholqr2_dist_workspace_bytes(self.ctx.handle, m, n, ctypes.byref(nbytes),
                                                                     ctypes.byref(ldg)), "cholqr2_dist workspace")
        g = torch.zeros((ldg.value, ldg.value), dtype=torch.float64, device=self.device)
        return {"ws": _dev.workspace(nbytes.value, self.device), "nbytes": nbytes.value, "G": g,
                "fallback": torch.zeros(1, dtype=torch.int32, device=self.device)}

    def cholqr2_dist(self, stage, a, r, state, flag=None):
        """One stage of the distributed Cholesky-QR2 of the shard ``a`` (in place)."""
        m, n = a.shape
        st = self.ctx.lib.pbq_cholqr2_dist(self.ctx.handle, int(stage), m, n, _dev.ptr(a), _dev.ld_of(a), _dev.ptr(r),
                                           _dev.ld_of(r), _dev.ptr(flag), _dev.ptr(state["G"]),
                                           _dev.ptr(state["fallback"]), _dev.ptr(state["ws"]), state["nbytes"],
                                           _dev.stream_ptr(self.device))
        self.ctx.check(st, "cholqr2_dist")


class DistributedPbpQlp:
    """One rank's part of a row-sharded PbP-QLP; all ranks call ``run``."""

    def __init__(self, n1, n2, d, q, rows, device=None, reorthonormalize=True, group=None, backend=None, chunks=None,
                 dist_qr="auto", exchange="nccl"):
        self.n1, self.n2, self.d, self.q = int(n1), int(n2), int(d), int(q)
        self.rows = list(rows)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if len(self.rows) != self.world + 1 or self.rows[0] != 0 or self.rows[-1] != n1:
            raise _exc.ParameterError("rows must be the G+1 shard offsets of [0, n1]")
        self.m = self.rows[self.rank + 1] - self.rows[self.rank]
        if self.m < self.d:
            raise _exc.ParameterError(f"each shard needs ≥ d={d} rows for the local TSQR leaf (rank {self.rank} has {self.m})")
        if not 1 <= self.d <= min(n1, n2):
            raise _exc.ParameterError(f"d must be in [1, {min(n1, n2)}], got {d}")
        self.reorthonormalize = bool(reorthonormalize)
        # allreduce pipelining depth for AᵀX (1 = one GEMM, then one allreduce)
        self.chunks = int(chunks) if chunks is not None else (4 if self.world > 1 else 1)
        if self.chunks < 1:
            raise _exc.ParameterError("chunks must be >= 1")
        self.be = backend if backend is not None else CudaBackend(device)
        be = self.be
        # AᵀX exchange: "nccl" — chunked GEMM + asynchronous allreduces;
        # "p2p" — the fused scatter-GEMM / slice reduce over peer memory
        if exchange not in ("nccl", "p2p"):
            raise _exc.ParameterError("exchange must be 'nccl' or 'p2p'")
        if exchange == "p2p" and not hasattr(be, "xchg_init"):
            raise _exc.ParameterError("this backend has no peer-memory exchange")
        self.exchange = exchange
        self.epoch = 0    # AᵀX exchanges
        self.ep_gram = 0  # Gram allreduces (p2p)
        self.ep_ag = 0    # all-gathers of orth(C) slices (p2p)
        self.poisoned = None  # set when a peer-memory wait timed out: the counters are no longer consistent
        self.xchg = be.xchg_init(self.n2, self.d, group) if exchange == "p2p" else None
        self._setup_c()
        self.exchange_note = exchange
        if self.xchg is not None:
            ok, why = self._p2p_self_check()
            if not ok:  # the whole group agreed (allreduce MIN): every rank falls back together
                self.xchg = None
                self.exchange = "nccl"
                self.epoch = self.ep_gram = self.ep_ag = 0
                self._setup_c()
                self.exchange_note = f"nccl (p2p self-check failed: {why})"
            else:
                self.exchange_note = f"p2p (self-check vs NCCL allreduce passed: {why})"
        self.Q = be.empty(self.m, self.d)          # A_g·P̄ → local Q_g → Q rows of this rank
        self.R = be.empty(self.d, self.d)
        self.Rloc = be.empty(self.d, self.d)
        self.stack = be.empty(self.world * self.d, self.d)
        self.Rs = be.empty(self.d, self.d)
        self.W = be.empty(self.d, self.d)
        self.Rt = be.empty(self.d, self.d)
        self.L = be.empty(self.d, self.d)
        self.P = be.empty(self.n2, self.d)
        self.Qtmp = be.empty(self.m, self.d)
        # [non-finite, sketch status, rank flags …, Cholesky-QR2 guard fired]
        self.flags = be.zeros_i32(2 * self.q + 4)
        self.force_fallback = False  # set by finish() for the re-run after a guard fired
        self.basis_orth = True       # intermediate orths: one Cholesky-QR pass (False: the full QR everywhere)
        self._last = None
        self.PHI = None
        # qr(A·P̄): distributed Cholesky-QR2 (one d×d allreduce per pass) with
        # the TSQR tree as its fallback, or the TSQR tree alone
        if dist_qr not in ("auto", "cholqr2", "tsqr"):
            raise _exc.ParameterError("dist_qr must be 'auto', 'cholqr2' or 'tsqr'")
        use_cq = dist_qr != "tsqr" and hasattr(be, "cholqr2_dist")
        if dist_qr == "cholqr2" and not use_cq:
            raise _exc.ParameterError("this backend has no distributed Cholesky-QR2")
        self.cq_state = be.cholqr2_dist_state(self.m, self.d) if use_cq else None
        self.tsqr_fallbacks = 0
        # orth(C) sharded over row slices (same distributed Cholesky-QR2, then an
        # all-gather of the slices) when every slice has ≥ d rows; else replicated
        self.c_state = (be.cholqr2_dist_state(self.slice_rows, self.d)
                        if use_cq and self.world > 1 and self.slice_rows >= self.d else None)
        self.orth_fallbacks = 0

    def _setup_c(self):
        """AᵀX partial → allreduced → P̄ (in place).  G·s rows (s = ⌈n2/G⌉, for
        p2p rounded to the 128-row tile) so that orth(C) can run on equal row
        slices; rows ≥ n2 stay zero."""
        if self.xchg is not None:
            self.slice_rows = self.xchg.S
            self.Cbuf = self.xchg.C[:, :self.d]
        else:
            self.slice_rows = -(-self.n2 // self.world)
            self.Cbuf = self.be.empty(self.world * self.slice_rows, self.d)
            ldc = self.Cbuf.stride(0)
            self.Cbuf.as_strided((self.Cbuf.shape[0], ldc), (ldc, 1)).zero_()  # incl. the even-ld pad column
        self.C = self.Cbuf[:self.n2]

    def _p2p_self_check(self, timeout_ms=2000):
        """Run one small AᵀX exchange, one Gram allreduce and one all-gather
        over peer memory with a short spin limit, and compare them with NCCL
        collectives of the same data.  Returns (ok, note), identical on every
        rank (the verdict is combined with an allreduce(MIN)); a mismatch or a
        timeout makes the caller fall back to the NCCL exchange."""
        import time

        be, x = self.be, self.xchg
        dev = x.land.device
        g = torch.Generator(device=dev)
        g.manual_seed(1000 + self.rank)
        k = 256  # rows of this rank's probe block
        a = torch.randn(k, self.n2, dtype=torch.float64, device=dev, generator=g)
        a = be.contiguous(a)
        xb = be.contiguous(torch.randn(k, self.d, dtype=torch.float64, device=dev, generator=g))
        ok, why = True, ""
        ctx = getattr(be, "ctx", None)
        if ctx is not None:
            ctx.set_p2p_timeout_ms(timeout_ms)
        t0 = time.perf_counter()
        try:
            # AᵀX: fused scatter GEMM + slice reduce + all-gather
            self.epoch += 1
            be.xchg_at_x(x, a, xb, self.n2, self.epoch)
            got = self.C.clone()
            ref = be.empty(self.n2, self.d)
            be.gemm_tn(a, xb, ref)
            ref = ref.contiguous()
            dist.all_reduce(ref, op=dist.ReduceOp.SUM, group=self.group)
            # Gram allreduce (push + slot-ordered sum)
            np_ = int(round(x.gram_slot ** 0.5))
            gram = torch.randn(np_, np_, dtype=torch.float64, device=dev, generator=g)
            gref = gram.clone()
            self.ep_gram += 1
            be.p2p_allreduce(x, gram, self.ep_gram)
            dist.all_reduce(gref, op=dist.ReduceOp.SUM, group=self.group)
            if dev.type == "cuda":
                torch.cuda.synchronize(dev)
            # every spin (tile count, done count, Gram pushes) ORs into the status word
            if int(x.status.item()):
                ok, why = False, "a peer did not arrive within %d ms" % timeout_ms
            else:
                scale = float(ref.abs().max()) or 1.0
                err = float((got - ref).abs().max()) / scale
                gerr = float((gram - gref).abs().max()) / (float(gref.abs().max()) or 1.0)
                if not (err <= 1e-12 and gerr <= 1e-12):
                    ok, why = False, f"results differ from NCCL (AᵀX rel err {err:.2e}, Gram {gerr:.2e})"
                else:
                    why = f"AᵀX rel err {err:.1e}, Gram {gerr:.1e}, {1e3 * (time.perf_counter() - t0):.0f} ms"
        except Exception as exc:  # noqa: BLE001  (e.g. an illegal peer address)
            ok, why = False, f"{type(exc).__name__}: {str(exc)[:100]}"
        finally:
            if ctx is not None:
                ctx.set_p2p_timeout_ms(20000)
        verdict = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(verdict, op=dist.ReduceOp.MIN, group=self.group)
        if ok and not int(verdict.item()):
            ok, why = False, "another rank's check failed"
        return ok, why

    def _check_usable(self):
        if self.poisoned:
            raise _exc.DeviceError(f"p2p exchange unusable after an earlier failure ({self.poisoned}); "
                                   "create a new DistributedPbpQlp")

    # -- collectives ---------------------------------------------------------
    def _chunk_bounds(self):
        """Row blocks of the n2×d result: multiples of the GEMM's 128-row tile
        (even starts keep the A column blocks 16-byte aligned)."""
        tiles = -(-self.n2 // 128)
        k = min(self.chunks, tiles)
        cuts = [128 * ((tiles * c) // k) for c in range(k)] + [self.n2]
        return [(cuts[c], cuts[c + 1]) for c in range(k) if cuts[c] < cuts[c + 1]]

    def _at_x(self, A_local, X, nonfinite=None):
        """self.C = Σ_g A_gᵀ·X_g with the allreduce of each row block
        overlapping the GEMM of the next one (or the fused p2p exchange)."""
        be = self.be
        C = self.C
        if self.xchg is not None:
            self.epoch += 1
            be.xchg_at_x(self.xchg, A_local, X, self.n2, self.epoch, nonfinite=nonfinite)
            return C
        ld = C.stride(0)
        padded = C.as_strided((C.shape[0], ld), (ld, 1))  # whole rows incl. the even-ld pad column
        handles = []
        for r0, r1 in self._chunk_bounds():
            be.gemm_tn(A_local[:, r0:r1], X, C[r0:r1], nonfinite=nonfinite)
            if self.world > 1 or self.chunks > 1:  # (world 1: exercises the pipeline)
                handles.append(dist.all_reduce(padded[r0:r1], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        for h in handles:
            h.wait()
        return C

    def _tsqr_(self, flag=None):
        """Distributed QR of the row-sharded self.Q (m_g × d) in place; R → self.R."""
        be = self.be
        be.qr_(self.Q, self.Rloc)
        rl = self.Rloc.contiguous()
        if dist.get_backend(self.group) == "nccl":
            gathered = torch.empty((self.world * self.d, self.d), dtype=rl.dtype, device=rl.device)
            dist.all_gather_into_tensor(gathered, rl, group=self.group)
        else:
            parts = [torch.empty_like(rl) for _ in range(self.world)]
            dist.all_gather(parts, rl, group=self.group)
            gathered = torch.cat(parts, 0)
        self.stack.copy_(gathered)
        be.qr_(self.stack, self.R, flag)  # replicated: same input on every rank
        qhat = self.stack[self.rank * self.d:(self.rank + 1) * self.d]
        be.gemm_nn(self.Q, be.contiguous(qhat), self.Qtmp)
        self.Q.copy_(self.Qtmp)

    def _sum_gram(self, g):
        """Allreduce(sum) of a d×d Gram: NCCL, or pushes into the peers' slots
        and a slot-ordered sum over symmetric memory (exchange="p2p")."""
        if self.xchg is None:
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)
            return
        self.ep_gram += 1
        self.be.p2p_allreduce(self.xchg, g, self.ep_gram)

    def _note_guard(self, st):
        """OR the call's guard flag into flags[-1] on the device (no sync)."""
        fb = self.flags[-1:]
        torch.maximum(fb, st["fallback"].to(fb.dtype), out=fb)

    def _cholqr2_stages(self, shard, r, st, flag, basis):
        """The distributed Cholesky-QR2 stages around their Gram allreduces.
        ``basis``: the result is only multiplied by A and orthonormalised again
        (an intermediate orth of the power iterations) — one pass and one Gram
        exchange (pbq_cholqr2_dist stage 3: shard ← Q·R₂, which leaves the next
        orth's Q factor unchanged)."""
        be = self.be
        be.cholqr2_dist(0, shard, r, st, flag)
        self._sum_gram(st["G"])
        if basis and self.basis_orth:
            be.cholqr2_dist(3, shard, r, st, flag)
        else:
            be.cholqr2_dist(1, shard, r, st, flag)
            self._sum_gram(st["G"])
            be.cholqr2_dist(2, shard, r, st, flag)
        self._note_guard(st)

    def _qr_sharded_(self, flag=None, basis=False):
        """QR of the row-sharded self.Q in place (R → self.R): distributed
        Cholesky-QR2 — local Gram, allreduce(sum) of the d×d Gram, replicated
        factor, local product, twice.  Its guard flag is noted on the device;
        the TSQR tree runs in the re-run that ``finish`` starts when it fired."""
        st = self.cq_state
        if st is None:
            return self._tsqr_(flag)
        if self.force_fallback:
            self.tsqr_fallbacks += 1
            return self._tsqr_(flag)
        self._cholqr2_stages(self.Q, self.R, st, flag, basis)

    def _orth_c_(self, flag, basis=False):
        """orth(C) in place, C replicated on every rank: each rank
        orthonormalizes its row slice by the distributed Cholesky-QR2 (two
        d×d allreduces), then the slices are all-gathered.  On a guard failure
        C is untouched everywhere and every rank runs the replicated QR."""
        st = self.c_state
        if st is None:
            return self.be.qr_(self.C, self.Rs, flag)
        if self.force_fallback:
            self.orth_fallbacks += 1
            return self.be.qr_(self.C, self.Rs, flag)
        be = self.be
        s0 = self.rank * self.slice_rows
        mine = self.Cbuf[s0:s0 + self.slice_rows]
        self._cholqr2_stages(mine, self.Rs, st, flag, basis)  # a fired guard left the slices untouched; finish() re-runs
        buf = self.Cbuf
        ld = buf.stride(0)
        whole = buf.as_strided((buf.shape[0], ld), (ld, 1))  # whole rows incl. the even-ld pad column
        part = whole[s0:s0 + self.slice_rows]
        if self.xchg is not None:
            self.ep_ag += 1
            self.be.p2p_allgather_rows(self.xchg, self.ep_ag)  # Cbuf is the symmetric C: peer stores
        elif dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(whole, part, group=self.group)  # in place: part is rank's chunk
        else:
            parts = [torch.empty_like(part) for _ in range(self.world)]
            dist.all_gather(parts, part.contiguous(), group=self.group)
            whole.copy_(torch.cat(parts, 0))

    # -- the algorithm ------------------------------------------------------
    def run(self, A_local, seed=0, phi_local=None):
        """Enqueue one factorization of this rank's rows (kernel-ready operand)."""
        self._check_usable()
        be = self.be
        d, q = self.d, self.q
        self._last = (A_local, seed, phi_local)
        self.flags.zero_()
        flags = self.flags
        if phi_local is None:
            self.PHI = be.gaussian(self.m, d, seed, self.rows[self.rank], status=flags[1:2])
        else:
            self.PHI = be.contiguous(phi_local)
        site = 2
        self._at_x(A_local, self.PHI, nonfinite=flags[0:1])
        if self.reorthonormalize:
            # every orth but the last is basis-only (its result feeds a pass
            # that is orthonormalised again; include/pbq.h: pbq_orth_basis)
            self._orth_c_(flags[site:site + 1], basis=(q >= 1))
            site += 1
            for it in range(q):
                be.gemm_nn(A_local, self.C, self.Q)
                self._qr_sharded_(flags[site:site + 1], basis=True)
                site += 1
                self._at_x(A_local, self.Q)
                self._orth_c_(flags[site:site + 1], basis=(it + 1 < q))
                site += 1
        else:
            for _ in range(q):
                be.gemm_nn(A_local, self.C, self.Q)
                self._at_x(A_local, self.Q)
            self._orth_c_(flags[site:site + 1])
        be.gemm_nn(A_local, self.C, self.Q)
        self._qr_sharded_()
        if hasattr(be, "second_stage"):
            be.second_stage(self.R, self.W, self.L)
        else:
            be.transpose(self.R, self.W)
            be.qr_(self.W, self.Rt)
            be.transpose(self.Rt, self.L, lower=True)
        be.gemm_nn(self.C, self.W, self.P)

    # -- CUDA graph of one sharded step --------------------------------------
    def capture(self, A_local, seed=0, phi_local=None):
        """Capture one ``run`` (kernels and NCCL collectives; every rank must
        call it) into a CUDA graph that ``replay`` relaunches with one call.
        The sketch seed is the captured one.  Only the NCCL exchange can be
        captured: the p2p exchange's spin targets are host-side epoch counts."""
        if self.xchg is not None:
            raise _exc.ParameterError("capture needs the NCCL exchange")
        dev = self.be.device
        self.run(A_local, seed, phi_local)  # warm: allocations, NCCL communicator, lazy loads
        self.finish()
        ctx = getattr(self.be, "ctx", None)
        launches0 = ctx.launch_count if ctx is not None else 0
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            self.run(A_local, seed, phi_local)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph_launches = (ctx.launch_count - launches0) if ctx is not None else 0
        self.graph = graph
        self.finish()
        return graph

    def replay(self):
        """Relaunch the captured step (``finish`` reads its flags as usual)."""
        self._check_usable()
        self.graph.replay()

    def finish(self, stacklevel=3):
        """Synchronise, raise / warn like the reference (every rank)."""
        # a non-finite entry in any shard fails every rank
        dist.all_reduce(self.flags[0:2], op=dist.ReduceOp.MAX, group=self.group)
        dist.all_reduce(self.flags[-1:], op=dist.ReduceOp.MAX, group=self.group)  # same on every rank anyway
        if self.xchg is not None and int(self.xchg.status.item()):
            # a late peer's increments could satisfy a later call's targets:
            # this exchange's counters are no longer consistent
            self.poisoned = "a peer did not arrive within the spin limit"
            raise _exc.DeviceError("p2p AᵀX exchange: a peer did not arrive within 20 s; the exchange is now "
                                   "unusable (create a new DistributedPbpQlp)")
        fl = self.flags.cpu().tolist()
        if fl[0]:
            raise _exc.MatrixInputError("a contains non-finite entries")
        if fl[1]:
            raise _exc.DeviceError("sketch generator overflow (internal error)")
        if fl[-1] and not self.force_fallback:
            # a Cholesky-QR2 guard fired (the same on every rank): redo the
            # factorization with the fallback in every QR
            self.force_fallback = True
            try:
                self.run(*self._last)
                return self.finish(stacklevel=stacklevel + 1)
            finally:
                self.force_fallback = False
        fl = fl[:-1]
        for f in fl[2:]:
            warn_rank(f, stacklevel=stacklevel + 1)
        return fl

    def factors(self):
        """(Q rows of this rank, L, P, R)."""
        return self.Q, self.L, self.P, self.R
