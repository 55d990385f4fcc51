"""pbp_qlp_multi_gpu at config-3 size with two gloo ranks sharing the one GPU
(validation of the launcher at scale, not a bench value): wall time of the
call, agreement with the single-GPU factors.   python tools/multigpu_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2103_07245_b200 import MultiGpuPool, pbp_qlp, pbp_qlp_multi_gpu, workloads

if __name__ == "__main__":
    dev = torch.device("cuda", 0)
    a = workloads.make("cfg3", 0, dev).cpu().numpy()
    one = pbp_qlp(a, 256, q=1, seed=3)
    t0 = time.perf_counter()
    two = pbp_qlp_multi_gpu(a, 256, q=1, seed=3, devices=[0, 0], backend="gloo")
    t = time.perf_counter() - t0
    def colerr(x, r):
        s = np.sign(np.sum(x * r, axis=0)); s[s == 0] = 1
        return float(np.max(np.linalg.norm(x * s - r, axis=0) / np.linalg.norm(r, axis=0)))
    l1, l2 = np.abs(np.diag(one.l)), np.abs(np.diag(two.l))
    print(f"2 gloo ranks on one GPU, 20000x10000 d=256 q=1: {t:.1f} s wall (process start-up, memory-mapped hand-over, "
          f"host-mediated collectives); vs single GPU: Q col err {colerr(two.q_basis, one.q_basis):.2e}, "
          f"P col err {colerr(two.p_basis, one.p_basis):.2e}, |diag L| rel err {float(np.max(np.abs(l1 - l2) / l1)):.2e}, "
          f"sketch bitwise equal: {bool(np.array_equal(one.sketch.test_matrix, two.sketch.test_matrix))}")
    t0 = time.perf_counter()
    with MultiGpuPool([0, 0], backend="gloo") as pool:
        t_start = time.perf_counter() - t0
        ts = []
        for i in range(4):
            t0 = time.perf_counter()
            f = pool.pbp_qlp(a, 256, q=1, seed=3 + i)
            ts.append(time.perf_counter() - t0)
    print(f"MultiGpuPool (same ranks): start-up {t_start:.1f} s, then per call " + ", ".join(f"{t:.2f}" for t in ts) +
          " s (hand-over of A through the memory-mapped file, staged H2D per rank, gloo collectives on one shared GPU)")
