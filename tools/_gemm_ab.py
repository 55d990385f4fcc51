import os, sys
sys.path.insert(0, "/root/repo")
from paper_2103_07245_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = sys.argv[1]
import torch
from paper_2103_07245_b200 import device as D
dev = torch.device("cuda", 0)
ctx = D.context(dev)
n1, n2, d = 20000, 10000, 256
a = D.empty_matrix(n1, n2, dev); a.normal_()
x = D.empty_matrix(n1, d, dev); x.normal_()
c = D.empty_matrix(n2, d, dev); c.normal_()
o1 = D.empty_matrix(n2, d, dev); o2 = D.empty_matrix(n1, d, dev)
ref1 = (a.T @ x); ref2 = a @ c
for name, fn, fl, ref, out in (("TN", lambda: D.gemm(ctx, a, x, True, out=o1), 2.0 * n1 * n2 * d, ref1, o1),
                     ("NN", lambda: D.gemm(ctx, a, c, False, out=o2), 2.0 * n1 * n2 * d, ref2, o2)):
    fn(); torch.cuda.synchronize()
    err = float((out - ref).abs().max() / ref.abs().max())
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 5)
    t = min(ts)
    print(f"{os.path.basename(_lib.LIB_PATH)} gemm {name}: {t:.3f} ms {fl / t / 1e9:.2f} TFLOP/s err {err:.1e}")
