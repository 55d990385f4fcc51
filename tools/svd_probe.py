"""Jacobi SVD core (pbq_jacobi_svd): sweeps, convergence, accuracy and time
per size and kernel.   python tools/svd_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D  # noqa: E402


def graded(n, L, decades, seed):
    rng = np.random.default_rng(seed)
    qa, _ = np.linalg.qr(rng.standard_normal((n, n)))
    qb, _ = np.linalg.qr(rng.standard_normal((L, n)))
    return (qa * np.logspace(0, -decades, n)) @ qb.T


def main():
    dev = torch.device("cuda", 0)
    ctx = D.context(dev)
    cases = [(256, 256, 8), (255, 300, 8), (255, 256, 8), (256, 300, 8), (255, 300, 0), (256, 512, 8), (200, 200, 8),
             (256, 256, 0), (128, 128, 8), (600, 600, 10)]
    for kernel in ("reg", "l2"):
        if kernel == "l2":
            os.environ["PBQ_JACOBI_L2"] = "1"
        for n, L, dec in cases:
            x = graded(n, L, dec, n + L)
            xt = D.as_kernel_operand(torch.from_numpy(x).to(dev))
            for acc in (True, False):
                s, y, g, st = D.jacobi_svd(ctx, xt, accumulate=acc)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                reps = 3
                for _ in range(reps):
                    D.jacobi_svd(ctx, xt, accumulate=acc)
                torch.cuda.synchronize()
                ms = (time.perf_counter() - t0) / reps * 1e3
                sw, nc = st.cpu().tolist()
                ref = np.linalg.svd(x, compute_uv=False)
                se = np.max(np.abs(s.cpu().numpy() - ref)) / ref[0]
                yo = np.abs(y.cpu().numpy() @ y.cpu().numpy().T - np.eye(n)).max()
                print(f"{kernel} n={n} L={L} dec={dec} acc={acc}: sweeps {sw} noconv {nc} |ds|/s0 {se:.1e} "
                      f"|YYᵀ-I| {yo:.1e} {ms:.3f} ms", flush=True)


def phases():
    """Where a register-kernel round goes (middle warp, clock64): rotate /
    send / wait cycles per round, via the debug hooks."""
    import ctypes
    dev = torch.device("cuda", 0)
    ctx = D.context(dev)
    fb = torch.zeros(1, dtype=torch.int32, device=dev)
    ph = torch.zeros(128, dtype=torch.int64, device=dev)
    bw = torch.zeros(1024, dtype=torch.int64, device=dev)
    ctx.lib.pbq_debug_qr_hooks(ctx.handle, ctypes.c_void_p(fb.data_ptr()), ctypes.c_void_p(ph.data_ptr()),
                               ctypes.c_void_p(bw.data_ptr()))
    for n, acc in ((256, True), (256, False), (128, True)):
        x = D.as_kernel_operand(torch.from_numpy(graded(n, n, 8, 2 * n)).to(dev))
        D.jacobi_svd(ctx, x, accumulate=acc, precondition=False)
        torch.cuda.synchronize()
        ph.zero_()
        D.jacobi_svd(ctx, x, accumulate=acc, precondition=False)
        torch.cuda.synchronize()
        rot, send, wait, rounds = ph.tolist()[40:44]
        rounds = max(rounds, 1)
        print(f"register kernel n={n} acc={acc}: per round rotate {rot / rounds:.0f}, send {send / rounds:.0f}, "
              f"wait+receive {wait / rounds:.0f} cycles ({rounds} rounds)", flush=True)
    ctx.lib.pbq_debug_qr_hooks(ctx.handle, None, None, None)


if __name__ == "__main__":
    if "--phases" in sys.argv:
        phases()
    else:
        main()
