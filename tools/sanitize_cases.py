"""Small invocations of every libpbq kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/sanitize_round.sh, one tool per
gpurun call).  Sizes are tiny: the sanitizers slow kernels by 10-1000x.

  python tools/sanitize_cases.py [case ...]

Cases: pipeline (config-1 shape PbP-QLP: sketch, TMA GEMMs with the TMEM
accumulator fold, the single-launch Cholesky-QR2 kernel, second stage),
chain (the multi-launch Cholesky-QR2: split-K Gram with its cooperative slice
sum, cooperative factor kernel, triangular products), householder (the blocked
cooperative Householder QR), shifted (shifted Cholesky-QR3 route),
cpqr_cluster / cpqr_grid (the pivot kernels), exchange (virtual-rank p2p
scatter GEMM / slice reduce / waits, G = 2), residual (fused residual GEMM),
svd (the preconditioned Jacobi SVD: QR chains, register cluster kernel,
GEMMs), svd_grid (the cooperative L2-resident Jacobi kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2103_07245_b200 import device as D  # noqa: E402
from paper_2103_07245_b200 import pbp_qlp, reconstruction_error  # noqa: E402


def pipeline(dev):
    from paper_2103_07245_b200 import workloads

    a = workloads.make_cfg1(0)
    f = pbp_qlp(a, 40, q=1, seed=1)
    print("pipeline ok", float(np.abs(np.diag(f.l))[0]))


def chain(dev):
    ctx = D.context(dev)
    ctx.set_qr_method(ctx.QR_CHOLQR_CHAIN)
    try:
        a = np.random.default_rng(8).standard_normal((900, 700))
        f = pbp_qlp(a, 160, q=1, seed=4)
    finally:
        ctx.set_qr_method(ctx.QR_AUTO)
    print("chain ok", float(np.abs(np.diag(f.l))[0]))


def householder(dev):
    ctx = D.context(dev)
    ctx.set_qr_method(ctx.QR_HOUSEHOLDER)
    try:
        a = np.random.default_rng(1).standard_normal((700, 48))
        f = pbp_qlp(a, 40, q=1, seed=2)
    finally:
        ctx.set_qr_method(ctx.QR_AUTO)
    print("householder ok", float(np.abs(np.diag(f.l))[0]))


def shifted(dev):
    rng = np.random.default_rng(3)
    m, n = 1200, 400
    g = rng.standard_normal((m, n)) * np.logspace(0, -9, n)
    t = D.as_kernel_operand(torch.from_numpy(g).to(dev))
    ctx = D.context(dev)
    D.householder_qr_(ctx, t, D.empty_matrix(n, n, dev))
    torch.cuda.synchronize()
    print("shifted ok")


def cpqr(dev, cluster=True):
    if not cluster:
        os.environ["PBQ_CPQR_NO_CLUSTER"] = "1"
    m = np.random.default_rng(4).standard_normal((96, 80)) * np.logspace(0, -6, 80)
    t = D.as_kernel_operand(torch.from_numpy(m).to(dev))
    p = D.cpqr_pivots(D.context(dev), t).cpu().numpy()
    os.environ.pop("PBQ_CPQR_NO_CLUSTER", None)
    print("cpqr ok", "cluster" if cluster else "grid", p[:5])


def exchange(dev):
    from paper_2103_07245_b200.distributed import shard_rows, virtual_exchanges

    ctx = D.context(dev)
    n1, n2, d, world = 400, 300, 40, 2
    rng = np.random.default_rng(5)
    a, x = rng.standard_normal((n1, n2)), rng.standard_normal((n1, d))
    xs = virtual_exchanges(n2, d, world, dev)
    rows = shard_rows(n1, world)
    for g in range(world):
        ag = D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(a[rows[g]:rows[g + 1]])).to(dev))
        xg = D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(x[rows[g]:rows[g + 1]])).to(dev))
        D.gemm_tn_scatter(ctx, ag, xg, xs[g])
    for r in range(world):
        D.xchg_reduce(ctx, xs[r], n2, d, D.xchg_expected_tiles(ctx, n2, d, xs[r].S, r, world))
    for r in range(world):
        D.xchg_wait(ctx, xs[r], 64 * world)
    torch.cuda.synchronize()
    err = np.abs(xs[0].C[:n2, :d].cpu().numpy() - a.T @ x).max()
    print("exchange ok", err)


def residual(dev):
    a = np.random.default_rng(6).standard_normal((300, 200))
    f = pbp_qlp(a, 30, q=0, seed=3)
    print("residual ok", reconstruction_error(a, f))


def svd(dev):
    if not hasattr(D, "jacobi_svd"):
        print("svd: not built")
        return
    m = torch.from_numpy(np.random.default_rng(7).standard_normal((70, 90))).to(dev)
    D.jacobi_svd(D.context(dev), D.as_kernel_operand(m))
    torch.cuda.synchronize()
    print("svd ok")


def svd_grid(dev):
    os.environ["PBQ_JACOBI_L2"] = "1"
    try:
        m = torch.from_numpy(np.random.default_rng(9).standard_normal((40, 50))).to(dev)
        D.jacobi_svd(D.context(dev), D.as_kernel_operand(m), precondition=False)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("PBQ_JACOBI_L2", None)
    print("svd_grid ok")


CASES = {"pipeline": pipeline, "chain": chain, "householder": householder, "shifted": shifted,
         "cpqr_cluster": lambda dev: cpqr(dev, True), "cpqr_grid": lambda dev: cpqr(dev, False),
         "exchange": exchange, "residual": residual, "svd": svd, "svd_grid": svd_grid}

if __name__ == "__main__":
    dev = torch.device("cuda", 0)
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name](dev)
