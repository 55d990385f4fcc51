"""One Jacobi SVD launch (n=256, L=256, accumulate) for ncu captures."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D  # noqa: E402

rng = np.random.default_rng(3)
qa, _ = np.linalg.qr(rng.standard_normal((256, 256)))
qb, _ = np.linalg.qr(rng.standard_normal((256, 256)))
x = (qa * np.logspace(0, -8, 256)) @ qb.T
xt = D.as_kernel_operand(torch.from_numpy(x).cuda())
ctx = D.context(torch.device("cuda", 0))
for _ in range(2):
    s, y, g, st = D.jacobi_svd(ctx, xt)
torch.cuda.synchronize()
print("sweeps", st.tolist())
