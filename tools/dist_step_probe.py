"""Per-rank cost of one row-sharded PbP-QLP step at a given shard size, on
one GPU (NCCL world of 1, so the collectives are real NCCL calls but local).

Emulates rank g of an N-GPU config-3 run: the shard has n1/N rows.  Reports
the GPU time per step (CUDA events, back-to-back steps) and the host time to
enqueue one step (the Python + C-ABI launch path); if the host time exceeds
the GPU time, the multi-GPU step is launch-bound.

    python tools/dist_step_probe.py [N] [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist


def main():
    n_emul = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    from paper_2103_07245_b200 import distributed as PD
    from paper_2103_07245_b200 import pbp_qlp_flops

    n1, n2, d, q = 20000, 10000, 256, 1
    m = n1 // n_emul
    a = torch.randn(m, n2, dtype=torch.float64, device=dev)
    run = PD.DistributedPbpQlp(m, n2, d, q, [0, m], dev, chunks=4)
    for i in range(3):
        run.run(a, seed=i)
        run.finish()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = []
    e0.record()
    for i in range(steps):
        t0 = time.perf_counter()
        run.run(a, seed=10 + i)
        host.append(time.perf_counter() - t0)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / steps
    host_ms = 1e3 * sorted(host)[len(host) // 2]
    fl = pbp_qlp_flops(n1, n2, d, q) / n_emul
    print(f"shard {m}x{n2} d={d} q={q} (config-3 rank of {n_emul}): GPU {gpu_ms:.3f} ms/step "
          f"({fl / gpu_ms / 1e9:.1f} TFLOP/s), host enqueue {host_ms:.3f} ms/step (median)")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
