"""Turn one round's GPU captures (gpurun_out/<tag>_*) into the tracked
summaries under profiles/:

  <tag>_launches_bench_cfg3.csv   raw ncu launch list of `python bench.py --steps 2 --warmup 1`
  <tag>_launch_shares.md           per-class share of one config-3 step
  <tag>_gemm_ncu.md                ncu --set full of the two A-pass GEMMs (TN, NN)
  <tag>_gemm_traffic.json          DRAM bytes per launch (read by bench.py for roofline.traffic)
  <tag>_cq_factor_ncu.md           ncu --set full of the Cholesky-QR factor kernel (pass 1, pass 2)
  <tag>_sketch_ncu.md              ncu --set full of the three sketch kernels
  <tag>_bench.json                 the bench line measured in the same session (no profiler)

    python tools/summarize_profiles.py r01c
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    return float(v.replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[unit]


def launch_shares(tag):
    src = os.path.join(OUT, f"{tag}_launches.csv")
    shutil.copy(src, os.path.join(PROF, f"{tag}_launches_bench_cfg3.csv"))
    lines = open(src).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = [r for r in csv.DictReader(lines[i:]) if r["Metric Name"] == "gpu__time_duration.sum"]

    def cls(n):
        if "gemm_f64_ring" in n or "gemm_f64_tma" in n:
            # template arguments: ring <T, BM, BN, BK, WM, WN, ST, CHECK, SPLIT, RESID>,
            # tma <T, BM, BN, WM, WN, ST, CHECK, SPLIT, RESID>
            args = [x.strip() for x in n[n.index("<") + 1:n.index(">")].split(",")]
            return "gemm_split" if args[-2] in ("1", "true") else "gemm"
        for k in ("cholqr_factor_kernel", "cholqr_gram_reduce", "qr_tall_kernel", "sketch_k1", "sketch_k2",
                  "sketch_k3", "transpose_kernel", "merge_flag_kernel", "pipeline_init_kernel", "copy_if_kernel",
                  "cholqr_mid_kernel", "cholqr_small_kernel"):
            if k in n:
                return k
        return "input-prep"

    seq = [(cls(r["Kernel Name"]), float(r["Metric Value"]) / 1e3, r["Grid Size"]) for r in rows]
    starts = [k for k, s in enumerate(seq) if s[0] == "sketch_k1"]
    step = seq[starts[1]:starts[2]]
    tot = sum(s[1] for s in step)
    groups = collections.OrderedDict()
    ntr = 0
    for name, us, grid in step:
        if name == "transpose_kernel":
            ntr += 1
        if name == "gemm" and us > 1000:
            key = "GEMM A-passes (gemm_f64_tma)"
        elif name == "gemm" and ntr == 2:
            key = "GEMM P = P̄·W (gemm_f64_tma)"
        elif name in ("gemm", "gemm_split", "cholqr_gram_reduce", "cholqr_factor_kernel", "qr_tall_kernel",
                      "copy_if_kernel", "cholqr_mid_kernel", "cholqr_small_kernel"):
            key = "QR ×5 (2 basis-only + 2 full Cholesky-QR2 chains, single-launch d×d; Householder / copy early-exit)"
        elif name.startswith("sketch"):
            key = "sketch (Philox4x64 + ziggurat, k1/k2/k3)"
        elif name == "input-prep":
            key = "torch kernels (seed writes of a graph replay)"
        else:
            key = "transposes + status init/merge"
        groups.setdefault(key, [0.0, 0])
        groups[key][0] += us
        groups[key][1] += 1
    md = [f"# {tag} launch list — share of one config-3 step", "",
          "Command (after the same command exited 0 without ncu): `ncu --metrics gpu__time_duration.sum "
          "--clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1` (raw list: "
          f"`{tag}_launches_bench_cfg3.csv`; one pipeline = the launches between consecutive `sketch_k1`).",
          "ncu serialises launches and flushes caches between them, so absolute times sit slightly above the",
          "in-stream CUDA-event times of bench.py; the shares are the comparable quantity.", "",
          "| class | launches | µs | share |", "|---|---|---|---|"]
    for k, (us, n) in groups.items():
        md.append(f"| {k} | {n} | {us:.0f} | {100 * us / tot:.1f}% |")
    md.append(f"| **total** | {len(step)} | {tot:.0f} | 100% |")
    bench = os.path.join(OUT, f"{tag}_bench.json")
    if os.path.exists(bench):
        line = [l for l in open(bench) if l.startswith("{")][-1]
        d = json.loads(line)
        r = d["roofline"]
        md += ["", f"bench.py in the same session (CUDA events, no profiler): step {d['ms_per_step']:.2f} ms = "
               f"{d['value'] / 1e3:.2f} TFLOP/s ({100 * d['value'] / 1e3 / 37.0:.1f}% of the 37.0 TFLOP/s FP64 peak); "
               f"GEMM {r['gemm_ms_per_step']:.2f} ms ({100 * r['gemm_ms_per_step'] / d['ms_per_step']:.1f}%, "
               f"{r['achieved']:.1f} TFLOP/s), QR {r['qr_ms_per_step']:.2f} ms, sketch {r['sketch_ms_per_step']:.2f} ms."]
        shutil.copy(bench, os.path.join(PROF, f"{tag}_bench.json"))
    md += ["", "Per launch (one step, in order):", "", "| # | kernel | grid | µs |", "|---|---|---|---|"]
    for j, (name, us, grid) in enumerate(step):
        md.append(f"| {j} | {name} | {grid} | {us:.1f} |")
    open(os.path.join(PROF, f"{tag}_launch_shares.md"), "w").write("\n".join(md) + "\n")


GEMM_KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
             ("dram__bytes_write.sum", "DRAM write"),
             ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active"),
             ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
             ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
             ("launch__registers_per_thread", "registers / thread"), ("launch__block_size", "block"),
             ("launch__grid_size", "grid"), ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
             ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts")]


def gemm(tag):
    reps = {"TN": os.path.join(OUT, f"{tag}_gemm_tn.ncu-rep"), "NN": os.path.join(OUT, f"{tag}_gemm_nn.ncu-rep")}
    vals = {k: raw(v) for k, v in reps.items()}
    md = [f"# {tag} ncu --set full: the DMMA GEMM on the config-3 A-passes", "",
          "`ncu --set full --import-source on --clock-control none -k regex:gemm_f64 --launch-skip {1,7} -c 1 "
          "python tools/gemm_probe.py` (TN = AᵀΦ 10000×256×20000, NN = A·P̄ 20000×256×10000), after the probe "
          "ran without ncu:", "", "```"] + open(os.path.join(OUT, f"{tag}_gemm_probe.txt")).read().strip().splitlines() + \
        ["```", "", "| metric | TN | NN |", "|---|---|---|"]
    for k, label in GEMM_KEYS:
        cells = []
        for t in ("TN", "NN"):
            h, u, rows = vals[t]
            cells.append(f"{rows[0][h.index(k)]} {u[h.index(k)]}" if k in h else "?")
        md.append(f"| {label} (`{k}`) | {cells[0]} | {cells[1]} |")
    traffic = {}
    for t in ("TN", "NN"):
        h, u, rows = vals[t]
        traffic[t] = sum(to_bytes(rows[0][h.index(k)], u[h.index(k)]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    avg = (traffic["TN"] + traffic["NN"]) / 2
    alg = 8.0 * (20000 * 10000 + 20000 * 256 + 10000 * 256)
    md += ["", f"DRAM traffic per launch: TN {traffic['TN'] / 1e9:.2f} GB, NN {traffic['NN'] / 1e9:.2f} GB "
           f"(average {avg / 1e9:.2f} GB) vs {alg / 1e9:.2f} GB algorithmic (A once + the thin operands once). "
           "The column tiles of one row tile run side by side in a CTA group of the stream-K schedule, so A "
           "leaves HBM about once per pass; the rest is thin-operand re-reads that miss L2."]
    open(os.path.join(PROF, f"{tag}_gemm_ncu.md"), "w").write("\n".join(md) + "\n")
    json.dump({"kernel": "gemm_f64_tma (config-3 A-passes)", "source": f"profiles/{tag}_gemm_ncu.md (ncu --set full)",
               "dram_bytes_per_launch": traffic, "dram_bytes_per_launch_avg": avg,
               "algorithmic_bytes_per_launch": alg}, open(os.path.join(PROF, f"{tag}_gemm_traffic.json"), "w"), indent=1)


def multi(tag, rep_name, title, labels, note):
    h, u, rows = raw(os.path.join(OUT, f"{tag}_{rep_name}.ncu-rep"))
    keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    md = [f"# {tag} ncu --set full: {title}", "", "| metric | " + " | ".join(labels[:len(rows)]) + " |",
          "|---|" + "---|" * len(rows[:len(labels)])]
    for k in keys:
        if k in h:
            md.append(f"| `{k}` | " + " | ".join(f"{r[h.index(k)]} {u[h.index(k)]}" for r in rows[:len(labels)]) + " |")
    md += ["", note]
    open(os.path.join(PROF, f"{tag}_{rep_name}_ncu.md"), "w").write("\n".join(md) + "\n")


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    launch_shares(tag)
    gemm(tag)
    if os.path.exists(os.path.join(OUT, f"{tag}_cq_factor.ncu-rep")):
        multi(tag, "cq_factor", "cholqr_factor_kernel (20000×256 QR)", ["pass 1 (blocked Cholesky + inverse)", "pass 2 (near-identity series)"],
              "Pass 1 is a chain of 8 block steps, each factoring a 32×32 diagonal block on one warp and ending "
              "with a grid barrier: latency-bound (few eligible warps, low issue). Pass 2 runs two parallel rounds "
              "of 32×32 block products.")
    if os.path.exists(os.path.join(OUT, f"{tag}_sketch.ncu-rep")):
        probe = open(os.path.join(OUT, f"{tag}_sketch_probe.txt")).read().strip()
        multi(tag, "sketch", "sketch kernels (20000×256 Φ)", ["k1 (Philox once + values)", "k2 (scan)", "k3 (compaction)"],
              "k1 is integer-multiply bound (Philox4x64-10: 64-bit multiplies); k3 is a memory-bound compaction.\n\n"
              "Probe (CUDA events): " + probe.replace("\n", "; "))
    print("wrote", sorted(f for f in os.listdir(PROF) if f.startswith(tag)))


if __name__ == "__main__":
    main()
