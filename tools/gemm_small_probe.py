"""Small-product GEMM latency (configs 1/2 passes and the second stage):
CUDA events over back-to-back launches, stream-ordered.

    PBQ_GEMM_MIN_UNITS=4 python tools/gemm_small_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D  # noqa: E402

SHAPES = [(1000, 40, 1000, False), (1000, 40, 1000, True), (4000, 100, 4000, False), (4000, 100, 4000, True),
          (100, 100, 100, False), (256, 256, 256, False), (10000, 256, 256, False)]


def main():
    dev = torch.device("cuda", 0)
    ctx = D.context(dev)
    tag = os.environ.get("PBQ_GEMM_MIN_UNITS", "1")
    for M, N, K, trans in SHAPES:
        a = D.empty_matrix(K if trans else M, M if trans else K, dev)
        a.normal_()
        b = D.empty_matrix(K, N, dev)
        b.normal_()
        c = D.empty_matrix(M, N, dev)
        for _ in range(5):
            D.gemm(ctx, a, b, trans_a=trans, out=c)
        torch.cuda.synchronize()
        reps = 50
        # device time: the launches captured in a CUDA graph (no host launch gaps)
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                D.gemm(ctx, a, b, trans_a=trans, out=c)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        print(f"min_units={tag} {'TN' if trans else 'NN'} M={M} N={N} K={K}: {us:.1f} us "
              f"({2.0 * M * N * K / us / 1e6:.2f} TFLOP/s)", flush=True)


if __name__ == "__main__":
    main()
