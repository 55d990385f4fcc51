"""Pinned host→device copy bandwidth (whole tensor vs chunked on 1/2 streams)."""
import time, torch
n = 20000 * 10000
h = torch.empty(n, dtype=torch.float64, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best
whole = t(lambda: d.copy_(h, non_blocking=True))
print(f"whole: {n*8/whole/1e9:.1f} GB/s ({whole*1e3:.1f} ms)")
streams = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    for chunks in (8, 32):
        def f():
            cs = n // chunks
            for i in range(chunks):
                with torch.cuda.stream(streams[i % ns]):
                    d[i*cs:(i+1)*cs].copy_(h[i*cs:(i+1)*cs], non_blocking=True)
        tt = t(f)
        print(f"streams {ns} chunks {chunks}: {n*8/tt/1e9:.1f} GB/s")
back = t(lambda: h.copy_(d, non_blocking=True))
print(f"d2h whole: {n*8/back/1e9:.1f} GB/s")
