import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2103_07245_b200 import device as D
dev = torch.device("cuda", 0)
ctx = D.context(dev)
for m, n in [(20000, 256), (256, 256)]:
    x0 = torch.randn(m, n, dtype=torch.float64, device=dev)
    x = D.empty_matrix(m, n, dev); r = D.empty_matrix(n, n, dev)
    for _ in range(3):
        x.copy_(x0); D.householder_qr_(ctx, x, r)
    torch.cuda.synchronize()
