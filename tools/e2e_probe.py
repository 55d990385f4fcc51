import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2103_07245_b200 import r_svd, cor_utv, pbp_qlp
from paper_2103_07245_b200 import device as D, workloads
from paper_2103_07245_b200.linalg import HostMatrix
dev = torch.device("cuda", 0)
a = workloads.make("cfg3", 0, dev).cpu().numpy()
def t(f, n=3):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)
print("r_svd e2e ms", t(lambda: r_svd(a, 256, q=1, seed=1)))
print("cor_utv e2e ms", t(lambda: cor_utv(a, 256, q=1, seed=1)))
print("pbp_qlp numpy e2e ms", t(lambda: pbp_qlp(a, 256, q=1, seed=1)))
ha = HostMatrix(a, "a")
print("to_device ms", t(lambda: ha.to_device(dev)))
A = ha.to_device(dev)
print("r_svd device-in ms", t(lambda: r_svd(A, 256, q=1, seed=1)))
u = torch.randn(20000, 256, dtype=torch.float64, device=dev)
print("u.cpu().numpy() ms", t(lambda: u.cpu().numpy()))
print("HostMatrix+all checks ms", t(lambda: HostMatrix(a, "a")))
