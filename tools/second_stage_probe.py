"""Time pbq_second_stage ((W, R̃) = qr(Rᵀ), L = tril(R̃ᵀ)) per d with CUDA events.

    python tools/second_stage_probe.py [d ...]      (PBQ_SECOND_STAGE=chain: the tall-QR chain)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2103_07245_b200 import device as D

dev = torch.device("cuda", 0)
ctx = D.context(dev)
for d in [int(x) for x in sys.argv[1:]] or [40, 64, 100, 128, 160, 256]:
    r = np.linalg.qr(np.random.default_rng(d).standard_normal((3 * d, d)))[1]
    rd = D.empty_matrix(d, d, dev)
    rd.copy_(torch.from_numpy(r))
    w, l = D.second_stage(ctx, rd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        D.second_stage(ctx, rd, w, l)
    e1.record()
    torch.cuda.synchronize()
    print(f"d={d}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
