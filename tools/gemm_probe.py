"""Time the FP64 DMMA GEMMs on the config-3 shapes (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_07245_b200 import device as D
dev = torch.device("cuda", 0)
ctx = D.context(dev)
n1, n2, d = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (20000, 10000, 256))]
a = D.empty_matrix(n1, n2, dev); a.normal_()
x = D.empty_matrix(n1, d, dev); x.normal_()
c = D.empty_matrix(n2, d, dev); c.normal_()
o1 = D.empty_matrix(n2, d, dev); o2 = D.empty_matrix(n1, d, dev)
for name, fn, fl in (("TN", lambda: D.gemm(ctx, a, x, True, out=o1), 2.0 * n1 * n2 * d),
                     ("NN", lambda: D.gemm(ctx, a, c, False, out=o2), 2.0 * n1 * n2 * d)):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): fn()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5
    print(f"gemm {name} {n1}x{n2}x{d}: {t:.3f} ms {fl / t / 1e9:.2f} TFLOP/s")
