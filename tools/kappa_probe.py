"""Condition number of every orth input of config 5 (d = 512, 1024; q = 2) and config 4:
which intermediate calls a looser basis-only guard would keep on the one-pass route.
(probe: torch.linalg.svdvals for κ₂)   python tools/kappa_probe.py"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D, workloads
dev = torch.device("cuda", 0)
ctx = D.context(dev)
def kappa(x):
    s = torch.linalg.svdvals(x.contiguous())
    return float(s[0] / s[-1])
for wl, d, q in (("cfg5", 512, 2), ("cfg5", 1024, 2), ("cfg4", 512, 1)):
    a = workloads.make_cfg5(0, dev) if wl == "cfg5" else workloads.make(wl, 0, dev)
    n1, n2 = a.shape
    phi = D.gaussian(ctx, n1, d, 0, dev)
    c = D.gemm(ctx, a, phi, trans_a=True)
    out = [f"orth(C0) {kappa(c):.2e}"]
    D.householder_qr_(ctx, c)
    for it in range(q):
        dm = D.gemm(ctx, a, c, trans_a=False)
        out.append(f"orth(D{it}) {kappa(dm):.2e}")
        D.householder_qr_(ctx, dm)
        c = D.gemm(ctx, a, dm, trans_a=True)
        out.append(f"orth(C{it + 1}) {kappa(c):.2e}")
        D.householder_qr_(ctx, c)
    dm = D.gemm(ctx, a, c, trans_a=False)
    out.append(f"qr(D) {kappa(dm):.2e}")
    print(wl, d, q, "kappa_2:", ", ".join(out), flush=True)
    del a, phi, c, dm
    torch.cuda.empty_cache()
