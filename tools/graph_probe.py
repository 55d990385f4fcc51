import sys, time
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2103_07245_b200 import PbpQlpPlan, workloads
dev = torch.device("cuda", 0)
for wl in ["cfg1", "cfg2", "cfg3"]:
    c = workloads.CONFIGS[wl]
    a = workloads.make(wl, 0, dev)
    plan = PbpQlpPlan(c["n1"], c["n2"], c["d"], c["q"], device=dev)
    plan.run(a, seed=0); plan.finish()
    q0 = plan.Q.clone()
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            plan.run(a, seed=0)
    except Exception as e:
        print(wl, "capture failed:", repr(e)[:300]); continue
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    print(wl, "replay equal:", torch.equal(plan.Q, q0))
    for mode in ("stream", "graph"):
        for _ in range(3):
            (g.replay() if mode == "graph" else plan.run(a, seed=0))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        for _ in range(20):
            (g.replay() if mode == "graph" else plan.run(a, seed=0))
        e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
        print(wl, mode, f"{e0.elapsed_time(e1)/20:.3f} ms/step (gpu)  {1e3*(t1-t0)/20:.3f} ms/step (host)")
