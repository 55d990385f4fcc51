import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2103_07245_b200 import device as D
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device('cuda', 0); ctx = D.context(dev)
rng = np.random.default_rng(0)
m = rng.standard_normal((n, n)) @ np.diag(np.exp(-np.arange(n) / (n / 10))) @ rng.standard_normal((n, n))
t = D.as_kernel_operand(torch.from_numpy(m).to(dev))
for _ in range(3):
    D.cpqr_pivots(ctx, t)
torch.cuda.synchronize()
print("ok")
