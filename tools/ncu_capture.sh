#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; one GPU, never multi-rank).
#   tools/ncu_capture.sh <tag> [kernel-regex ...]
# 1) launch list with per-launch device time (cold-cache, serialised: compare SHARES)
# 2) one --set full capture per kernel regex (default: the three hot kernels)
set -u
TAG=${1:-r01}; shift || true
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
BATCH=${ICL_NCU_BATCH:-8}  # the bench default launch (8 x 4096^2 per filter): traffic is read from THE timed launch shape
BENCH="python bench.py --steps 2 --warmup 3 --batch $BATCH --no-e2e --no-cpu-baseline --no-tune --no-small --no-16k"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/launches_bench.log 2>&1
echo "launch list rc=$?"
REGEXES=("$@")
if [ ${#REGEXES[@]} -eq 0 ]; then REGEXES=(nlm_sym sep_stream harris_shfl); fi
for K in "${REGEXES[@]}"; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $OUT/full_$K $BENCH > $OUT/full_$K.log 2>&1
  echo "full $K rc=$?"
done
