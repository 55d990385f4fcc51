#!/usr/bin/env bash
# FP64 peak with its clock record: run the DMMA/DFMA
# microbenchmark while nvidia-smi samples SM clocks and throttle reasons.
#   gpurun -- 'bash tools/fp64_peak_round.sh <tag>'  →  gpurun_out/<tag>_fp64_peak.jsonl
set -u
TAG=${1:?tag}
O=gpurun_out
mkdir -p $O
B=tools/microbench/fp64_peak
[ -x $B ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/fp64_peak.cu -o $B
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,power.draw,temperature.gpu \
  --format=csv,noheader -lms 100 > $O/${TAG}_fp64_clocks.csv 2>/dev/null &
SMI=$!
sleep 0.5
for rep in 1 2 3; do $B; done > $O/${TAG}_fp64_peak.jsonl 2>&1
kill $SMI 2>/dev/null
wait $SMI 2>/dev/null
python - "$O/${TAG}_fp64_clocks.csv" "$O/${TAG}_fp64_peak.jsonl" <<'PY'
import json, statistics, sys
rows = [r.split(", ") for r in open(sys.argv[1]).read().strip().splitlines() if r]
mhz = [float(r[1].split()[0]) for r in rows if len(r) > 3 and r[1].split()[0].replace(".", "").isdigit()]
mx = [float(r[2].split()[0]) for r in rows if len(r) > 3 and r[2].split()[0].replace(".", "").isdigit()]
reasons = sorted({r[3] for r in rows if len(r) > 3})
rec = {"clocks": {"sm_mhz_median": statistics.median(mhz) if mhz else None, "sm_mhz_min": min(mhz) if mhz else None,
                  "sm_max_mhz": max(mx) if mx else None, "throttle_reasons_bitmasks": reasons, "samples": len(mhz)}}
open(sys.argv[2], "a").write(json.dumps(rec) + "\n")
print(json.dumps(rec))
PY
cat $O/${TAG}_fp64_peak.jsonl
