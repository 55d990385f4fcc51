#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_cases.py, ONE tool per gpurun call:
#   gpurun -- 'bash tools/sanitize_round.sh <tag> memcheck|racecheck|synccheck'
# Summaries land in gpurun_out/<tag>_<tool>.txt (copied to profiles/ after review).
set -u
TAG=${1:?tag}
TOOL=${2:?tool}
O=gpurun_out
mkdir -p $O
python tools/sanitize_cases.py > $O/${TAG}_${TOOL}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
EXTRA=""
[ "$TOOL" = memcheck ] && EXTRA="--leak-check no"
for c in pipeline chain householder shifted cpqr_cluster cpqr_grid exchange residual svd svd_grid; do
  echo "=== case $c ($TOOL)" >> $O/${TAG}_${TOOL}.txt
  timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --report-api-errors no --print-limit 20 \
    python tools/sanitize_cases.py $c >> $O/${TAG}_${TOOL}.txt 2>&1
  echo "exit $?" >> $O/${TAG}_${TOOL}.txt
done
grep -E "^=== case|ERROR SUMMARY|RACECHECK SUMMARY|exit " $O/${TAG}_${TOOL}.txt
