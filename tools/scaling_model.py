"""Strong-scaling model from one GPU (no multi-GPU box was available in
rounds 1-2).  For N in {1, 2, 4, 8}, run the row-sharded driver
(distributed.DistributedPbpQlp) of ONE rank of an N-GPU job on a shard of
n1/N rows, in a world-1 NCCL group — the collectives are real NCCL calls on
the n2×d and d×d buffers of the full problem, only their transfer is local —
captured as a CUDA graph exactly as bench.py does for N > 1, and timed as
graph replays.  The per-rank time T_N is the N-GPU step without the
inter-GPU transfer; the model adds the transfer at a stated NVLink bus
bandwidth:

    comm_N = (q+1)·allreduce(n2·d·8 B) + (4 + 2q)·allreduce(d²·8 B)
             (two Gram exchanges per full Cholesky-QR2, one per basis-only intermediate orth)
    allreduce(b) = 2·(N−1)/N · b / BW_bus,  BW_bus = 600 GB/s (NVLink 5 ring,
    conservative vs. 900 GB/s per direction)

and reports predicted speed-ups T_1 / (T_N + comm_N).  A model, not a
measurement: the driver's SCALE run is the measurement.

    python tools/scaling_model.py [--workload cfg4|cfg3] [--steps K]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

SHAPES = {"cfg3": (20000, 10000, 256, 1), "cfg4": (200000, 8192, 512, 1)}
BW_BUS = 600e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4", choices=sorted(SHAPES))
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    from paper_2103_07245_b200 import distributed as PD
    from paper_2103_07245_b200 import pbp_qlp_flops

    n1, n2, d, q = SHAPES[args.workload]
    flops = pbp_qlp_flops(n1, n2, d, q)
    t1 = None
    for n in (1, 2, 4, 8):
        m = n1 // n
        a = torch.randn(m, n2, dtype=torch.float64, device=dev)
        run = PD.DistributedPbpQlp(m, n2, d, q, [0, m], dev)
        for i in range(2):
            run.run(a, seed=i)
            run.finish()
        run.capture(a, seed=7)
        for _ in range(2):
            run.replay()
        run.finish()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            run.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        # per-class split from a stream-ordered repeat with events around every kernel
        ctx = getattr(run.be, "ctx", None)
        by_class = None
        if ctx is not None:
            ctx.profile_begin(capacity=4096)
            run.run(a, seed=11)
            torch.cuda.synchronize()
            by_class = {k: round(v[0], 3) for k, v in ctx.profile_end().items()}
            run.finish()
        if n == 1:
            t1 = ms
        big = (q + 1) * n2 * d * 8
        # Gram allreduces: two per full distributed Cholesky-QR2 (the last orth(C) and qr(A·P̄)),
        # one per basis-only intermediate orth (2q of them when q ≥ 1; pbq_cholqr2_dist stage 3)
        small = (2 * 2 + 2 * q if q >= 1 else 2 * 2) * d * d * 8
        comm_ms = 0.0 if n == 1 else 1e3 * 2 * (n - 1) / n * (big + small) / BW_BUS
        line = {"workload": args.workload, "n1": n1, "n2": n2, "d": d, "q": q, "N": n, "shard_rows": m,
                "per_rank_ms": round(ms, 3), "per_rank_tflops": round(flops / n / ms / 1e9, 2),
                "comm_model_ms": round(comm_ms, 3), "predicted_ms": round(ms + comm_ms, 3),
                "predicted_speedup": round(t1 / (ms + comm_ms), 2), "bw_bus_gbs": BW_BUS / 1e9,
                "graph": "captured", "class_ms_stream_ordered": by_class, "note": "one rank of an N-GPU job on one GPU (world-1 NCCL); model, not a measurement"}
        print(json.dumps(line), flush=True)
        del run, a
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
