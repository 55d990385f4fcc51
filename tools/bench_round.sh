#!/usr/bin/env bash
# The bench lines of one GPU session (run on the box):  bash tools/bench_round.sh <tag>
# Default line (config 3, e2e + CPU baseline), the reference arm, configs 1/2/4,
# the config-5 d-sweep and the sibling paths.
set -u
TAG=${1:?tag}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${TAG}_bench_full.json 2> $O/${TAG}_bench_full.err
python bench.py --impl reference > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err
for w in cfg1 cfg2 cfg4; do
  python bench.py --workload $w --no-cpu-baseline > $O/${TAG}_${w}.json 2> $O/${TAG}_${w}.err
done
for q in 0 2; do for d in 64 128 256 512 1024; do
  python bench.py --workload cfg5 --d $d --q $q --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
    >> $O/${TAG}_cfg5_sweep.jsonl 2>> $O/${TAG}_cfg5_sweep.err
done; done
for p in r_svd cor_utv; do
  python bench.py --path $p --no-cpu-baseline > $O/${TAG}_${p}.json 2> $O/${TAG}_${p}.err
done
echo done
