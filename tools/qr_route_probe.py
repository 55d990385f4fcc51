"""Which QR route each configuration takes (stats [done, Householder fallbacks, pass 2 by the series,
done by the shifted route]) and the per-class split of one factorization.   python tools/qr_route_probe.py"""
import sys, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D, workloads, PbpQlpPlan
dev = torch.device("cuda", 0)
for wl, d, q in (("cfg4", 512, 1), ("cfg5", 512, 0), ("cfg5", 1024, 0), ("cfg3", 256, 1)):
    a = workloads.make(wl, 0, dev) if wl != "cfg5" else workloads.make_cfg5(0, dev)
    n1, n2 = a.shape
    plan = PbpQlpPlan(n1, n2, d, q, device=dev)
    ctx = plan.ctx
    stats = torch.zeros(4, dtype=torch.int32, device=dev)
    ctx.cholqr_stats(stats)
    plan.run(a, seed=1); plan.finish()
    torch.cuda.synchronize()
    ctx.profile_begin(4096)
    plan.run(a, seed=2); plan.finish()
    cls = ctx.profile_end()
    print(wl, d, q, "stats [done, hh fallbacks, series, shifted] =", stats.tolist(), {k: round(v[0], 2) for k, v in cls.items()}, flush=True)
    ctx.cholqr_stats(None)
    del a, plan
    torch.cuda.empty_cache()
