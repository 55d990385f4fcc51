#!/usr/bin/env bash
# One GPU session's captures and their summaries (tools/summarize_profiles.py <tag>).
# Run on the box:  gpurun -- 'bash tools/profile_round.sh <tag>'
# Every ncu command runs only after the same command exited 0 without ncu.
# The four .ncu-rep files together exceed what gpurun copies back (64 MiB), so
# they are summarised on the box: the summaries land in gpurun_out/prof/ (copy
# them into profiles/) and the reports are deleted unless KEEP_REPS=1.
set -u
TAG=${1:?tag}
O=gpurun_out
mkdir -p $O
NCU="ncu --clock-control none"
python bench.py --no-e2e --no-cpu-baseline > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err || exit 1
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1 || exit 1
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/${TAG}_ncu_launches.log 2>&1
python tools/gemm_probe.py > $O/${TAG}_gemm_probe.txt 2>&1 || exit 1
$NCU --set full --import-source on -k regex:gemm_f64 --launch-skip 1 -c 1 -f -o $O/${TAG}_gemm_tn \
  python tools/gemm_probe.py > $O/${TAG}_ncu_gemm_tn.log 2>&1
$NCU --set full --import-source on -k regex:gemm_f64 --launch-skip 7 -c 1 -f -o $O/${TAG}_gemm_nn \
  python tools/gemm_probe.py > $O/${TAG}_ncu_gemm_nn.log 2>&1
python tools/_cq_one.py > /dev/null 2>&1 || exit 1
$NCU --set full --import-source on -k regex:cholqr_factor_kernel --launch-skip 4 -c 2 -f -o $O/${TAG}_cq_factor \
  python tools/_cq_one.py > $O/${TAG}_ncu_cq.log 2>&1
python tools/sketch_probe.py > $O/${TAG}_sketch_probe.txt 2>&1 || exit 1
$NCU --set full --import-source on -k regex:sketch_k -c 3 -f -o $O/${TAG}_sketch \
  python tools/sketch_probe.py > $O/${TAG}_ncu_sketch.log 2>&1
python tools/summarize_profiles.py $TAG > $O/${TAG}_summarize.log 2>&1
mkdir -p $O/prof && cp profiles/${TAG}_* $O/prof/
[ "${KEEP_REPS:-0}" = 1 ] || rm -f $O/${TAG}_*.ncu-rep
echo done
