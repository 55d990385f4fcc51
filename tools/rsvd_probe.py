"""r_svd per-stage times at config 3 (and the reference's n=2000, d=600
timing case): CUDA events around each stage of one call.
   python tools/rsvd_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D, workloads  # noqa: E402
from paper_2103_07245_b200.rsvd import r_svd  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ctx = D.context(dev)
    a = workloads.make_cfg3(0, dev)
    for _ in range(2):
        r_svd(a, 256, q=1, seed=1)
    torch.cuda.synchronize()
    for rep in range(3):
        ctx.profile_begin(4096)
        t0 = time.perf_counter()
        r_svd(a, 256, q=1, seed=2 + rep)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        cls = ctx.profile_end()
        print(f"cfg3 r_svd wall {wall:.2f} ms; by class {cls}", flush=True)
    rh = D.empty_matrix(256, 256, dev)
    rh.copy_(torch.triu(torch.randn(256, 256, dtype=torch.float64, device=dev)))
    st = torch.zeros(2, dtype=torch.int32, device=dev)
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.jacobi_svd(ctx, rh, status=st)
        e1.record()
        torch.cuda.synchronize()
        print(f"jacobi 256x256 triangular: {e0.elapsed_time(e1):.3f} ms, sweeps {st.tolist()}", flush=True)
    rng = np.random.default_rng(0)
    b = rng.standard_normal((2000, 2000))
    for q in (0, 1, 2):
        r_svd(b, 600, q=q, seed=0)
        ts = []
        for t in range(5):
            t0 = time.perf_counter()
            r_svd(b, 600, q=q, seed=1 + t)
            ts.append(time.perf_counter() - t0)
        print(f"n=2000 d=600 q={q}: median {np.median(ts) * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
