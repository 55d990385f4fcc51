"""Cholesky-QR2 vs Householder QR on the device: accuracy against numpy's
LAPACK QR (sign-fixed like linalg.py:96-103), which path ran, and timing.

    python tools/cholqr_probe.py [MxN ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2103_07245_b200 import device as D

shapes = [(20000, 256), (10000, 256), (256, 256), (1000, 40), (4000, 100), (333, 65), (700, 48), (8192, 512),
          (50, 1), (64, 64), (100, 33)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
dev = torch.device("cuda", 0)
ctx = D.context(dev)
stats = torch.zeros(4, dtype=torch.int32, device=dev)
ctx.cholqr_stats(stats)


def ref_qr(a):
    q, r = np.linalg.qr(a)
    s = np.sign(np.diag(r))
    s[s == 0] = 1
    return q * s, (r * s[:, None])


def run(method, x0, reps=5):
    ctx.set_qr_method(method)
    m, n = x0.shape
    x = D.empty_matrix(m, n, dev)
    r = D.empty_matrix(n, n, dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ts = []
    for i in range(reps + 2):
        x.copy_(x0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.householder_qr_(ctx, x, r, rank_flag=flag)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return x.cpu().numpy(), r.cpu().numpy(), int(flag.item()), min(ts)


def case(name, a_np):
    m, n = a_np.shape
    x0 = torch.from_numpy(a_np).to(dev)
    qr_, rr_ = ref_qr(a_np)
    out = []
    for method in (0, 3, 1):  # auto (single-launch kernel where it applies), the 7-launch chain, Householder
        stats.zero_()
        q, r, flag, t = run(method, x0)
        st = stats.tolist()
        eq = np.max(np.linalg.norm(q - qr_, axis=0) / np.linalg.norm(qr_, axis=0))
        er = np.linalg.norm(r - rr_) / np.linalg.norm(rr_) if np.linalg.norm(rr_) > 0 else 0.0
        orth = np.linalg.norm(q.T @ q - np.eye(n))
        out.append(f"{ {0: 'auto', 3: 'chain', 1: 'hh'}[method]:5s} {t*1e3:8.1f}us eq={eq:.1e} er={er:.1e} "
                   f"orth={orth:.1e} flag={flag} stats={st}")
    print(f"{name:>22s}: " + " | ".join(out), flush=True)


rng = np.random.default_rng(0)
for m, n in shapes:
    case(f"{m}x{n}", rng.standard_normal((m, n)))
# graded columns (κ ~ 1e4) and ill-conditioned (κ ~ 1e12 → fallback)
a = rng.standard_normal((4000, 128)) * np.logspace(0, -4, 128)
case("graded 1e-4", a)
u, _ = np.linalg.qr(rng.standard_normal((4000, 128)))
v, _ = np.linalg.qr(rng.standard_normal((128, 128)))
case("kappa 1e12", (u * np.logspace(0, -12, 128)) @ v.T)
b = rng.standard_normal((2000, 96))
b[:, 50] = b[:, 3]
case("rank deficient", b)
case("zero", np.zeros((300, 40)))
ctx.cholqr_stats(None)

if os.environ.get("CQ_PHASES"):
    import ctypes
    fb = torch.zeros(1, dtype=torch.int32, device=dev)
    ph = torch.zeros(128, dtype=torch.int64, device=dev)
    bw = torch.zeros(1024, dtype=torch.int64, device=dev)
    ctx.lib.pbq_debug_qr_hooks(ctx.handle, ctypes.c_void_p(fb.data_ptr()), ctypes.c_void_p(ph.data_ptr()),
                               ctypes.c_void_p(bw.data_ptr()))
    ctx.set_qr_method(0)
    names = ["chol+inv", "items", "barrier", "final"]
    for m, n in [(20000, 256), (10000, 256), (256, 256), (8192, 512)]:
        x = D.empty_matrix(m, n, dev)
        x.normal_()
        r = D.empty_matrix(n, n, dev)
        D.householder_qr_(ctx, x, r)
        torch.cuda.synchronize()
        ph.zero_()
        x.normal_()
        D.householder_qr_(ctx, x, r)
        torch.cuda.synchronize()
        v = [t / 1e3 for t in ph.tolist()[:8]]
        print(f"{m}x{n} factor phases (us): pass1 " + ", ".join(f"{a}={b:.1f}" for a, b in zip(names, v[:4])) +
              " | pass2 " + ", ".join(f"{a}={b:.1f}" for a, b in zip(names, v[4:8])))
        cl = [t / 1e3 for t in ph.tolist()[8:]]
        if any(cl):
            for c in range((n + 31) // 32):
                print(f"   cluster CTA {c:2d}: " + ", ".join(
                    f"{a}={b:.1f}" for a, b in zip(["A", "bar1", "B", "bar2", "C"], cl[5 * c:5 * c + 5])))
    names_s = ["gram1+bar", "reduce1+bar", "factor1", "tri+gram2+bar", "reduce2+bar", "factor2", "R", "final tri"]
    for m, n in [(1000, 40), (4000, 100), (64, 64), (100, 33), (50, 1), (256, 100)]:
        x = D.empty_matrix(m, n, dev)
        x.normal_()
        r = D.empty_matrix(n, n, dev)
        D.householder_qr_(ctx, x, r)
        torch.cuda.synchronize()
        ph.zero_()
        x.normal_()
        D.householder_qr_(ctx, x, r)
        torch.cuda.synchronize()
        v = [t / 1e3 for t in ph.tolist()[16:24]]
        print(f"{m}x{n} single-launch phases (us): " + ", ".join(f"{a}={b:.1f}" for a, b in zip(names_s, v)))
    names_m = ["gram1+sums", "factor1", "Q1", "gram2+sums", "factor2", "Q"]
    for m, n in [(256, 256), (200, 160), (1000, 200)]:
        x = D.empty_matrix(m, n, dev)
        x.normal_()
        r = D.empty_matrix(n, n, dev)
        D.householder_qr_(ctx, x, r)
        torch.cuda.synchronize()
        ph.zero_()
        x.normal_()
        D.householder_qr_(ctx, x, r)
        torch.cuda.synchronize()
        v = [t / 1e3 for t in ph.tolist()[24:30]]
        print(f"{m}x{n} mid-size single-launch phases (us): " + ", ".join(f"{a}={b:.1f}" for a, b in zip(names_m, v)))
    ctx.lib.pbq_debug_qr_hooks(ctx.handle, None, None, None)
