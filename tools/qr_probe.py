"""Time the device Householder QR on given shapes (CUDA events)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_07245_b200 import device as D

shapes = [(10000, 256), (20000, 256), (256, 256), (1000, 40), (4000, 100), (8192, 512), (25000, 512)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
dev = torch.device("cuda", 0)
ctx = D.context(dev)
for m, n in shapes:
    x = D.empty_matrix(m, n, dev)
    x.normal_()
    src = x.clone()
    r = D.empty_matrix(n, n, dev)
    for _ in range(2):
        x.copy_(src)
        D.householder_qr_(ctx, x, r)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        x.copy_(src)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.householder_qr_(ctx, x, r)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    fl = 4.0 * m * n * n - 4.0 * n ** 3 / 3
    print(f"qr {m}x{n}: {t:.3f} ms  {fl / t / 1e6:.1f} GFLOP/s  ({t * 1e3 / n:.2f} us/column)")

if os.environ.get("QR_PHASES"):
    import ctypes
    names = ["gram1+bar", "reduce1+chol1", "pass2+gram2+bars", "chol2+small", "pass3", "fallback", "wpartial+bar",
             "reduce+bar", "update", "R/zero+bar", "orgqr W+bars", "orgqr update+gen", "chol2", "Qp", "LU", "T+M1", "oq:V1T", "oq:vform", "oq:wpart", "oq:bar1", "oq:reduce"]
    fb = torch.zeros(1, dtype=torch.int32, device=dev)
    ph = torch.zeros(24, dtype=torch.int64, device=dev)
    bw = torch.zeros(1024, dtype=torch.int64, device=dev)
    ctx.lib.pbq_debug_qr_hooks(ctx.handle, ctypes.c_void_p(fb.data_ptr()), ctypes.c_void_p(ph.data_ptr()),
                               ctypes.c_void_p(bw.data_ptr()))
    for m, n in shapes:
        x = D.empty_matrix(m, n, dev)
        x.normal_()
        ph.zero_()
        bw.zero_()
        D.householder_qr_(ctx, x, D.empty_matrix(n, n, dev))
        torch.cuda.synchronize()
        w = bw[:148].double() / 1e3
        nz = w[w > 0]
        print(f"  barrier spin per CTA (us): min {nz.min():.1f} median {nz.median():.1f} max {nz.max():.1f} "
              f"argmin {int(torch.argmin(torch.where(w > 0, w, torch.full_like(w, 1e18))))}")
        tot = ph.sum().item()
        print(f"{m}x{n}: fallbacks={fb.item()} total {tot/1e3:.1f} us: " +
              ", ".join(f"{nm}={v/1e3:.1f}" for nm, v in zip(names, ph.tolist()) if v))
    ctx.lib.pbq_debug_qr_hooks(ctx.handle, None, None, None)
