import time, numpy as np, torch
a = np.random.default_rng(0).standard_normal((20000, 10000))
rt = torch.cuda.cudart()
d = torch.empty((20000, 10000), dtype=torch.float64, device="cuda")
t = torch.from_numpy(a)
for rep in range(3):
    t0 = time.perf_counter()
    r = rt.cudaHostRegister(t.data_ptr(), t.numel() * 8, 0)
    t1 = time.perf_counter()
    d.copy_(t, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(t.data_ptr())
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms (rc {r}), copy {1e3*(t2-t1):.1f} ms, unregister {1e3*(t3-t2):.1f} ms")
