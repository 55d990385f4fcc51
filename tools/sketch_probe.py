"""Time the device sketch generator (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_07245_b200 import device as D
dev = torch.device("cuda", 0)
ctx = D.context(dev)
for rows, cols in [(20000, 256), (200000, 512)]:
    out = D.empty_matrix(rows, cols, dev)
    D.gaussian(ctx, rows, cols, 7, dev, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        D.gaussian(ctx, rows, cols, 7, dev, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"sketch {rows}x{cols}: {e0.elapsed_time(e1) / 5:.3f} ms")
