"""Orthogonality of the Householder kernel's Q on ill-conditioned inputs (A/B:
PBQ_QR_SLOW_PANELS=1 forces the column-by-column panel path)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D
dev = torch.device("cuda", 0)
ctx = D.context(dev)
ctx.set_qr_method(1)
rng = np.random.default_rng(0)
for m, n, logk in ((129, 129, 13), (256, 256, 13), (129, 129, 8), (1000, 129, 13), (2000, 200, 13), (500, 96, 13)):
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    x = (u * np.logspace(0, -logk, n)) @ v.T
    t = D.as_kernel_operand(torch.from_numpy(x).to(dev))
    r = D.empty_matrix(n, n, dev)
    D.householder_qr_(ctx, t, r)
    q = t.cpu().numpy()
    ql, _ = np.linalg.qr(x)
    print(f"{m}x{n} k=1e{logk}: |QtQ-I| {np.abs(q.T @ q - np.eye(n)).max():.1e}  LAPACK {np.abs(ql.T @ ql - np.eye(n)).max():.1e}", flush=True)
