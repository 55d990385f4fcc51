#!/usr/bin/env python3
"""PbP-QLP benchmark (BASELINE.json metric: GFLOP/s and % FP64 roofline at
20000×10000, d=256, q=1; 1/2/4/8-GPU scaling).

One *step* = one full PbP-QLP factorization (device sketch, 2q+2 passes over
A, all QRs, L and P) of the synthetic config-3 matrix resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload cfg3] [--no-cpu-baseline] [--no-e2e]

For N > 1 launch under torchrun (one rank per GPU, NCCL); A is row-sharded
across ranks (strong scaling: the same A is split N ways), timing is the max
over ranks of CUDA-event time.  ``--impl reference`` times the reference's CPU
implementation (the oracle port of pbpqlp.pbp_qlp, numpy/OpenBLAS on all host
cores) on the same workload; under torchrun only rank 0 runs it.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.17  # measured DMMA.8x8x4 peak at 1965 MHz, profiles/r02_fp64_peak.jsonl (clock record inside)
FP64_PEAK_SOURCE = "measured: tools/microbench/fp64_peak.cu DMMA m8n8k4, 16 warps/SM, on this pool's B200 at a median 1965 MHz SM clock with no throttle reason (tools/fp64_peak_round.sh, profiles/r02_fp64_peak.jsonl); MEASURED_PEAKS.json has no FP64 entry"
METRIC = "PbP-QLP GFLOP/s and % FP64 roofline at 20000x10000, d=256; 1/2/4/8 GPU scaling"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time stream-ordered launches instead of replays of the captured CUDA graph (N = 1)")
    ap.add_argument("--d", type=int, default=None, help="override the workload's d (config-5 d-sweep)")
    ap.add_argument("--q", type=int, default=None, help="override the workload's q")
    ap.add_argument("--path", default="pbp_qlp", choices=["pbp_qlp", "r_svd", "cor_utv"],
                    help="r_svd / cor_utv: the sibling randomized paths (SURVEY §8 f3), single GPU")
    ap.add_argument("--exchange", default="nccl", choices=["p2p", "nccl"],
                    help="N > 1 AᵀX exchange: nccl (default) = chunked GEMM + asynchronous ncclAllReduce; p2p = the "
                         "fused scatter-GEMM / slice reduce over NVLink peer memory (self-checked against NCCL at "
                         "init, falls back to nccl on mismatch or timeout)")
    ap.add_argument("--no-cfg4", action="store_true",
                    help="skip the extra config-4 (200000x8192, d=512, q=1) timing carried in the default line")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: validates the N>1 code path with ranks sharing GPUs (host-mediated "
                         "collectives); its timings are not bench values")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")


def reference_impl(path="pbp_qlp"):
    """The CPU implementation the baseline times: the STOCK reference
    (``pbpqlp`` installed unmodified under baseline/_ref by
    tools/install_reference.sh) when present — kind "reference" — else the
    oracle port of its call sequence (oracle/pbp_qlp_oracle.py, kind "port")."""
    if os.path.isfile(os.path.join(REF_INSTALL, "pbpqlp", "__init__.py")):
        if REF_INSTALL not in sys.path:
            sys.path.insert(0, REF_INSTALL)
        import pbpqlp

        fn = getattr(pbpqlp, path)
        return fn, "reference", f"stock pbpqlp {pbpqlp.__version__}.{path} from baseline/_ref"
    from oracle import pbp_qlp_oracle as O

    fn = {"pbp_qlp": O.oracle_pbp_qlp, "r_svd": O.oracle_r_svd, "cor_utv": O.oracle_cor_utv}[path]
    return fn, "port", f"oracle port oracle/pbp_qlp_oracle.py:oracle_{path} (reference call sequence)"


def host_info():
    """CPU model, numpy and BLAS build of the host the CPU baseline ran on."""
    import numpy as np

    info = {"numpy": np.__version__, "cores_available": cpu_threads()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["cpu_model"] = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info

        info["threadpools"] = [{k: tp.get(k) for k in ("user_api", "internal_api", "version", "num_threads",
                                                       "threading_layer", "architecture")}
                               for tp in threadpool_info()]
    except Exception as exc:  # noqa: BLE001
        info["threadpools"] = f"unavailable: {exc}"
    return info


def time_cpu_oracle(a_host, wl, seed, steps, budget_s=None):
    """Time the reference's CPU path on all host cores: the stock pbpqlp when
    installed (kind "reference"), else the oracle port (kind "port")."""
    import warnings

    from threadpoolctl import threadpool_limits

    from paper_2103_07245_b200 import pbp_qlp_flops

    fn, kind, prov = reference_impl("pbp_qlp")
    cores = cpu_threads()
    n1, n2, d, q = wl["n1"], wl["n2"], wl["d"], wl["q"]
    a = a_host
    sample = f"full {n1}x{n2} d={d} q={q} factorization per step"
    times = []
    with threadpool_limits(limits=cores), warnings.catch_warnings():
        warnings.simplefilter("ignore")
        t0 = time.perf_counter()
        fn(a, d, q=q, seed=seed)  # discarded warm-up (cli.py:393-415 protocol)
        first = time.perf_counter() - t0
        if budget_s is not None and first * steps > budget_s:
            rows = max(d, int(n1 * budget_s / (first * steps * 1.2)))
            a = a_host[:rows]
            n1 = rows
            sample = f"row sample {rows}x{n2} of the {wl['n1']}x{n2} matrix, d={d} q={q}, per step"
        for i in range(steps):
            t0 = time.perf_counter()
            fn(a, d, q=q, seed=seed + 1 + i)
            times.append(time.perf_counter() - t0)
    f = pbp_qlp_flops(n1, n2, d, q)
    med = statistics.median(times)
    return {"value": f / med / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": kind,
            "sample": sample + f" ({len(times)} timed after 1 discarded, median {med:.3f} s, "
                               f"mean {statistics.mean(times):.3f} s; {prov}; numpy/OpenBLAS on {cores} threads)",
            "seconds": med, "times": times, "host": host_info()}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path (the stock pbpqlp from
    baseline/_ref, else the oracle port) on rank 0 only."""
    if rank != 0:
        return
    import numpy as np
    import torch

    from paper_2103_07245_b200 import workloads

    wl = workload(args)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    a = workloads.make(args.workload, args.seed, dev).cpu().numpy()
    res = time_cpu_oracle(a, wl, args.seed, args.steps, budget_s=180.0)
    line = {
        "metric": METRIC, "value": res["value"], "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["seconds"] * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, wl, world),
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample", "host")},
        "e2e": {"value": res["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload(args):
    """BASELINE config, with optional --d / --q overrides (the config-5 sweep)."""
    from paper_2103_07245_b200 import workloads

    wl = dict(workloads.CONFIGS[args.workload])
    if args.d is not None:
        wl["d"] = args.d
    if args.q is not None:
        wl["q"] = args.q
    return wl


def config_dict(args, wl, world):
    return {
        "workload": f"{args.workload}: A {wl['n1']}x{wl['n2']} fp64 synthetic (BASELINE config), d={wl['d']}, q={wl['q']}, seeded device sketch",
        "n1": wl["n1"], "n2": wl["n2"], "d": wl["d"], "q": wl["q"], "seed": args.seed,
        "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
        "l2": "inputs larger than L2 (A is 1.6 GB vs 126 MB L2)" if wl["n1"] * wl["n2"] * 8 > 126e6 else "A fits L2",
    }


def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2103_07245_b200 import PbpQlpPlan, pbp_qlp, pbp_qlp_flops, workloads
    from paper_2103_07245_b200 import device as D

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wl = workload(args)
    n1, n2, d, q = wl["n1"], wl["n2"], wl["d"], wl["q"]
    flops = pbp_qlp_flops(n1, n2, d, q)

    if world > 1:
        from paper_2103_07245_b200 import distributed as PD

        a_full = workloads.make(args.workload, args.seed, dev)
        rows = PD.shard_rows(n1, world)
        a = a_full[rows[rank]:rows[rank + 1]].contiguous()
        del a_full
        torch.cuda.empty_cache()
        # p2p needs GPUs of their own (its waits span ranks): never with the
        # gloo validation mode, where ranks share a GPU
        runner, exchange_note = make_runner(args, PD, n1, n2, d, q, rows, dev)
        step = lambda s: runner.run(a, seed=s)  # noqa: E731
        finish = runner.finish
        ctx = D.context(dev)
    else:
        a = workloads.make(args.workload, args.seed, dev)
        plan = PbpQlpPlan(n1, n2, d, q, device=dev)
        step = lambda s: plan.run(a, seed=s)  # noqa: E731
        finish = plan.finish
        ctx = plan.ctx

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(args.seed + i)
        finish()
    # one GPU: the whole factorization is captured once as a CUDA graph and
    # each timed step is a replay with a new seed (every kernel runs again).
    # N > 1 with the NCCL exchange: the sharded step (kernels + NCCL
    # collectives) is captured the same way, replayed with the captured seed;
    # the p2p exchange stays stream-ordered (its spin targets are host-side
    # epoch counters baked into the launches).
    graph = not args.no_graph
    graph_note = None
    if graph and world == 1:
        plan.capture(a)
        for i in range(args.warmup):
            plan.replay(args.seed + 50 + i)
        finish()
    elif graph:
        graph_note = try_capture_dist(runner, a, args, finish)
        graph = graph_note == "captured"
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    barrier()
    launches0 = ctx.launch_count
    if not graph:
        ctx.profile_begin(capacity=64 * (2 * q + 8) * args.steps)  # events around every kernel, same stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        if graph and world == 1:
            plan.replay(args.seed + 100 + i)
        elif graph:
            runner.replay()
        else:
            step(args.seed + 100 + i)
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if graph:
        launches = (plan.graph_launches if world == 1 else runner.graph_launches) * args.steps
        finish()
        # per-kernel-class times: CUDA events around every launch of the same
        # steps, stream-ordered (events cannot sit between the graph's nodes)
        barrier()
        ctx.profile_begin(capacity=64 * (2 * q + 8) * args.steps)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        for i in range(args.steps):
            step(args.seed + 100 + i)
        p1.record()
        torch.cuda.synchronize()
        by_class = ctx.profile_end()
        instrumented_ms = p0.elapsed_time(p1) / args.steps
    else:
        by_class = ctx.profile_end()
        launches = ctx.launch_count - launches0
        instrumented_ms = None
    finish()
    ms = e0.elapsed_time(e1) / args.steps

    # ---- reconstruction check of the last timed step (outside the timed
    # region): ‖A − QLPᵀ‖_F/‖A‖_F by the fused one-pass residual kernel
    check = None
    if world == 1:
        from paper_2103_07245_b200 import QlpFactors, reconstruction_error

        f = QlpFactors(plan.Q, plan.L, plan.P, None)
        check = {"recon_rel_err": reconstruction_error(a, f),
                 "method": "pbq_residual_fro (fused GEMM + residual epilogue, one pass over A)"}
    else:
        qg, l, p, _ = runner.factors()
        sums = D.residual_fro(ctx, a, qg, l, p)  # this shard's ‖A_g − Q_g L Pᵀ‖², ‖A_g‖²
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        r2, a2 = sums.tolist()
        check = {"recon_rel_err": (r2 / a2) ** 0.5,
                 "method": "pbq_residual_fro per row shard (fused GEMM + residual epilogue) + allreduce(sum)"}
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = flops / (ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (FP64 DMMA GEMM, 2q+2 launches/step),
    # from the CUDA events recorded around each launch inside the timed region
    roof = None
    if rank == 0:
        traffic = gemm_traffic(args.workload) if world == 1 else {"bytes": None, "source": None}
        gemm_ms, gemm_n = by_class["gemm"]
        big = 2 * q + 2  # A-passes per step; the P̄·W product is 2·n2·d² flops
        m_loc = n1 if world == 1 else (n1 * (rank + 1)) // world - (n1 * rank) // world  # this rank's rows
        fl_pass = 2.0 * m_loc * n2 * d
        fl_small = 2.0 * n2 * d * d + (0.0 if world == 1 else (q + 1) * 2.0 * m_loc * d * d)  # + TSQR Q·Q̂
        fl_total = args.steps * (big * fl_pass + fl_small)
        achieved = fl_total / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        roof = {
            "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS if achieved else None, "traffic": traffic["bytes"],
            "traffic_unit": "bytes per launch (DRAM read + write)", "traffic_source": traffic["source"],
            "algorithmic_bytes_per_launch": 8.0 * (m_loc * n2 + m_loc * d + n2 * d),
            "kernel": "gemm_f64_tma (C=A^T X and D=A X, FP64 DMMA.8x8x4, TMA-staged)" + ("" if world == 1 else
                      f", rank 0's row shard ({m_loc} rows); AᵀX exchange: {exchange_note}"),
            "per_launch_flop": fl_pass, "launches_per_step": gemm_n / args.steps,
            "gemm_ms_per_step": gemm_ms / args.steps,
            "gemm_share_of_step": gemm_ms / args.steps / (instrumented_ms or ms),
            "qr_ms_per_step": by_class["qr"][0] / args.steps, "sketch_ms_per_step": by_class["sketch"][0] / args.steps,
            "other_ms_per_step": by_class["other"][0] / args.steps,
            "step_frac_of_peak": value / 1e3 / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE,
            "measured": ("CUDA events around every launch on the launch stream, in a stream-ordered repeat of the "
                         f"timed steps ({instrumented_ms:.3f} ms/step with the events; the timed steps are CUDA-graph "
                         "replays)") if instrumented_ms is not None else
                        "CUDA events around every launch on the launch stream, inside the timed region",
        }

    # ---- end to end through the public API with host (pinned) input
    e2e = None
    if not args.no_e2e and world > 1:
        # each rank: its pinned host shard → device, the sharded factorization,
        # its Q rows (and on rank 0 the replicated L, P, R) back to the host;
        # the step time is the max over ranks
        a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        a_host.copy_(a)
        del a
        torch.cuda.empty_cache()
        ts = []
        for i in range(max(3, min(args.steps, 10)) + 1):
            barrier()
            t0 = time.perf_counter()
            a_dev = D.as_kernel_operand(a_host.to(dev, non_blocking=True))
            runner.run(a_dev, seed=args.seed + 200 + i)
            runner.finish()
            qg, l, p, r = runner.factors()
            outs = [qg.cpu()] + ([l.cpu(), p.cpu(), r.cpu()] if rank == 0 else [])
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            del a_dev
            if i > 0:  # the first call is the warm-up
                ts.append(float(dt.item()))
        t_e2e = statistics.median(ts)
        d2h = sum(x.numel() * 8 for x in outs)
        e2e = {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(a_host.numel() * 8),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": t_e2e * 1e3,
               "input": "pinned host row shard per rank (bytes: rank 0's)", "max_over_ranks": True}
    if not args.no_e2e and world == 1:
        a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        a_host.copy_(a)
        del plan
        torch.cuda.synchronize()
        f = pbp_qlp(a_host, d, q=q, seed=args.seed)  # warm
        ts = []
        for i in range(max(3, min(args.steps, 10))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = pbp_qlp(a_host, d, q=q, seed=args.seed + 200 + i)
            ts.append(time.perf_counter() - t0)
        t_e2e = statistics.median(ts)
        d2h = sum(x.numel() * 8 for x in (f.q_basis, f.l, f.p_basis, f.first_stage_r)) + 4 * (2 * q + 2)
        e2e = {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(n1 * n2 * 8),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": t_e2e * 1e3, "input": "pinned host torch tensor"}
        # the reference's own calling convention: a (pageable) numpy array in,
        # numpy factors out — staged through the plan's pinned ring
        a_np = np.array(a_host.numpy())  # a pageable copy
        pbp_qlp(a_np, d, q=q, seed=args.seed)  # warm (plan cache, pinned ring)
        ts = []
        for i in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            f = pbp_qlp(a_np, d, q=q, seed=args.seed + 300 + i)
            ts.append(time.perf_counter() - t0)
        t_np = statistics.median(ts)
        e2e["numpy"] = {"value": flops / t_np / 1e9, "unit": "GFLOP/s", "ms_per_step": t_np * 1e3,
                        "h2d_bytes_per_step": int(n1 * n2 * 8), "d2h_bytes_per_step": int(d2h),
                        "input": "pageable numpy float64 array (the reference's calling convention), staged through "
                                 "a pinned ring overlapped with the H2D DMA and the first pass"}
        del a_np, f
        from paper_2103_07245_b200 import clear_plan_cache

        clear_plan_cache()
        torch.cuda.empty_cache()

    # ---- config 4 (the north star's scaling shape) timed in the same run, so
    # the driver's N = 1 and N > 1 lines both carry it
    cfg4 = None
    if args.workload == "cfg3" and not args.no_cfg4 and args.d is None and args.q is None:
        a = None  # release config 3's A (the step closures hold the name, not the tensor)
        torch.cuda.empty_cache()
        cfg4 = time_cfg4(args, world, rank, dev, barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        a_np = a_host.numpy() if e2e is not None else workloads.make(args.workload, args.seed, dev).cpu().numpy()
        res = time_cpu_oracle(a_np, wl, args.seed, steps=3, budget_s=60.0)
        cpu = {k: res[k] for k in ("value", "unit", "cores", "kind", "sample", "host")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, wl, world),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "check": check,
        }
        if cfg4 is not None:
            line["cfg4"] = cfg4
        if graph_note is not None:
            line["graph"] = graph_note
        if world > 1:
            line["exchange"] = exchange_note
        if world > 1 and args.dist_backend != "nccl":
            line["validation_only"] = f"{args.dist_backend} collectives, ranks sharing GPUs: not a bench value"
        print(json.dumps(line), flush=True)


def make_runner(args, PD, n1, n2, d, q, rows, dev):
    """The row-sharded driver with the requested AᵀX exchange.  "p2p" (one
    GPU per rank only) checks itself against NCCL at init and falls back."""
    exchange = args.exchange
    if exchange == "p2p" and args.dist_backend != "nccl":
        raise SystemExit("--exchange p2p needs --dist-backend nccl (one GPU per rank)")
    try:
        runner = PD.DistributedPbpQlp(n1, n2, d, q, rows, dev, exchange=exchange)
        note = runner.exchange_note
    except Exception as exc:  # noqa: BLE001  symmetric memory unavailable: the NCCL exchange
        runner = PD.DistributedPbpQlp(n1, n2, d, q, rows, dev, exchange="nccl")
        note = f"nccl (p2p unavailable: {type(exc).__name__}: {str(exc)[:120]})"
    return runner, note


def try_capture_dist(runner, a, args, finish):
    """Capture the sharded step as a CUDA graph (NCCL exchange only); returns
    "captured" or why it stays stream-ordered."""
    if runner.exchange != "nccl":
        return "stream-ordered: the p2p exchange's spin targets are host-side epochs"
    import torch.distributed as dist

    if dist.get_backend() != "nccl":  # the gloo validation mode: host-mediated collectives cannot be captured
        return "stream-ordered: gloo collectives are host-mediated (validation mode)"
    try:
        runner.capture(a, seed=args.seed + 50)
        for _ in range(args.warmup):
            runner.replay()
        finish()
        return "captured"
    except Exception as exc:  # noqa: BLE001
        import torch

        torch.cuda.synchronize()
        # the capture's invalidation error is still this thread's CUDA
        # last-error: clear it, or the next stream-ordered launch reports it
        getattr(runner.be, "ctx", None) and runner.be.ctx.clear_error()
        return f"stream-ordered: capture failed ({type(exc).__name__}: {str(exc)[:120]})"


def time_cfg4(args, world, rank, dev, barrier):
    """Config 4 (200000x8192 fp64, d=512, q=1) — the north star's ≥6x-at-8-GPU
    shape — timed like the main line: N = 1 as CUDA-graph replays, N > 1
    row-sharded (same A split N ways; max over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2103_07245_b200 import PbpQlpPlan, pbp_qlp_flops, workloads

    n1, n2, d, q = 200000, 8192, 512, 1
    flops = pbp_qlp_flops(n1, n2, d, q)
    steps = max(3, min(args.steps, 5))
    a = workloads.make_cfg4(args.seed, dev)
    note = None
    if world > 1:
        from paper_2103_07245_b200 import distributed as PD

        rows = PD.shard_rows(n1, world)
        a = a[rows[rank]:rows[rank + 1]].contiguous()
        torch.cuda.empty_cache()
        runner, note = make_runner(args, PD, n1, n2, d, q, rows, dev)
        runner.run(a, seed=args.seed)
        runner.finish()
        gnote = try_capture_dist(runner, a, args, runner.finish) if not args.no_graph else "stream-ordered"
        step = runner.replay if gnote == "captured" else (lambda: runner.run(a, seed=args.seed))
        fin = runner.finish
    else:
        plan = PbpQlpPlan(n1, n2, d, q, device=dev)
        plan.run(a, seed=args.seed)
        plan.finish()
        plan.capture(a)
        for i in range(args.warmup):
            plan.replay(args.seed + 1 + i)
        plan.finish()
        gnote = "captured"
        it = iter(range(10**9))
        step = lambda: plan.replay(args.seed + 100 + next(it))  # noqa: E731
        fin = plan.finish
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    fin()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = flops / (ms * 1e-3) / 1e9
    out = {"workload": f"cfg4: A {n1}x{n2} fp64 synthetic (BASELINE config 4), d={d}, q={q}, seeded device sketch"
                       + ("" if world == 1 else f", row-sharded x{world} (strong scaling)"),
           "ms_per_step": ms, "value": value, "unit": "GFLOP/s", "steps": steps,
           "frac_of_fp64_peak": value / 1e3 / FP64_PEAK_TFLOPS, "graph": gnote}
    if note is not None:
        out["exchange"] = note
    return out


def run_sibling(args):
    """--path r_svd | cor_utv: the sibling randomized paths on
    the same kernels, same JSON contract, on one GPU."""
    import numpy as np
    import torch

    from paper_2103_07245_b200 import workloads
    from paper_2103_07245_b200 import device as D
    from paper_2103_07245_b200.rsvd import r_svd, r_svd_flops
    from paper_2103_07245_b200.utv import cor_utv, cor_utv_flops

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    wl = workload(args)
    n1, n2, d, q = wl["n1"], wl["n2"], wl["d"], wl["q"]
    k = min(n1, d)
    if args.path == "r_svd":
        fn, passes = r_svd, 2 * q + 2
        flops = r_svd_flops(n1, n2, d, q)
        d2h = 8 * (n1 + n2 + 1) * k
    else:  # cor_utv with the exact core (2q + 3 passes), reference defaults
        fn, passes = cor_utv, 2 * q + 3
        flops = cor_utv_flops(n1, n2, d, q)
        d2h = 8 * (n1 * k + k * d + n2 * d)
    a = workloads.make(args.workload, args.seed, dev)
    ctx = D.context(dev)
    for i in range(args.warmup):
        fn(a, d, q=q, seed=args.seed + i)
    torch.cuda.synchronize()
    # host-orchestrated paths (Python between launches), so the value is timed
    # in a clean pass; an identical second pass carries the per-launch events
    # (GEMM roofline) and the nvidia-smi clock sampling.
    launches0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        fn(a, d, q=q, seed=args.seed + 100 + i)  # one flag read per call (host sync), as the API does
    e1.record()
    torch.cuda.synchronize()
    launches = ctx.launch_count - launches0
    ms = e0.elapsed_time(e1) / args.steps
    sampler = ClockSampler(0)
    sampler.start()
    time.sleep(0.2)
    ctx.profile_begin(capacity=64 * (2 * q + 12) * args.steps)
    for i in range(args.steps):
        fn(a, d, q=q, seed=args.seed + 100 + i)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    clocks["sampled"] = "during an identical second timed pass"
    by_class = ctx.profile_end()
    value = flops / (ms * 1e-3) / 1e9
    gemm_ms, gemm_n = by_class["gemm"]
    fl_gemm = args.steps * (passes * 2.0 * n1 * n2 * d)
    roof = {"bound": "tensor", "achieved": fl_gemm / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None,
            "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "traffic": None,
            "kernel": f"gemm_f64_tma (the {passes} A-passes)", "gemm_ms_per_step": gemm_ms / args.steps,
            "qr_ms_per_step": by_class["qr"][0] / args.steps, "sketch_ms_per_step": by_class["sketch"][0] / args.steps,
            "step_frac_of_peak": value / 1e3 / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE}
    if roof["achieved"]:
        roof["frac"] = roof["achieved"] / FP64_PEAK_TFLOPS
    cpu = None
    if not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits

        a_np = a.cpu().numpy()
        import warnings

        ref_fn, kind, prov = reference_impl(args.path)
        with threadpool_limits(limits=cpu_threads()), warnings.catch_warnings():
            warnings.simplefilter("ignore")
            ref_fn(a_np, d, q=q, seed=args.seed)  # discarded warm-up
            t0 = time.perf_counter()
            ref_fn(a_np, d, q=q, seed=args.seed + 1)
            sec = time.perf_counter() - t0
        cpu = {"value": flops / sec / 1e9, "unit": "GFLOP/s", "cores": cpu_threads(), "kind": kind,
               "sample": f"one full {n1}x{n2} d={d} q={q} {args.path} after one discarded ({sec:.3f} s; {prov}; "
                         f"numpy/OpenBLAS)", "host": host_info()}
    # e2e: numpy in, numpy out through the public function
    e2e = None
    if not args.no_e2e:
        a_host = a.cpu().numpy()
        fn(a_host, d, q=q, seed=args.seed)
        t0 = time.perf_counter()
        fn(a_host, d, q=q, seed=args.seed + 1)
        sec = time.perf_counter() - t0
        e2e = {"value": flops / sec / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(a_host.nbytes),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": sec * 1e3, "input": "numpy host array (pageable)"}
    line = {"metric": f"{args.path} GFLOP/s at {n1}x{n2}, d={d}, q={q}", "value": value, "unit": "GFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, wl, 1), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clocks, "path": args.path}
    print(json.dumps(line), flush=True)


def gemm_traffic(workload):
    """DRAM bytes per A-pass launch of the GEMM from the newest committed
    `ncu --set full` capture (profiles/*_gemm_traffic.json, config 3 only)."""
    import glob

    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "*_gemm_traffic.json")))
    if workload != "cfg3" or not files:
        return {"bytes": None, "source": None}
    with open(files[-1]) as f:
        rec = json.load(f)
    return {"bytes": rec["dram_bytes_per_launch_avg"], "source": os.path.relpath(files[-1], os.path.dirname(os.path.abspath(__file__)))}


def main():
    args = parse()
    world, rank, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.impl == "reference":
            if rank == 0:
                run_reference(args, world, rank)
            return
        if args.dist_backend == "gloo":  # validation mode: ranks may share a GPU
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            run_ours(args, world, rank, local)
        finally:
            dist.destroy_process_group()
        return
    if args.path in ("r_svd", "cor_utv"):
        run_sibling(args)
    elif args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
