#!/bin/bash
# Profile recipe (run under gpurun from the repo root; one GPU).  Writes to gpurun_out/.
#   1. launch list of the bench command (per-launch device time, cold-cache, serialised)
#   2. one full ncu capture of the top kernel (monitor_kernel_*) for DRAM traffic/stalls
set -e
TAG=${1:-r01}
WL=${2:-C2}
EXTRA=${3:-}          # e.g. "--nan-mode mask"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}_${WL}.csv \
    python bench.py --workload $WL $EXTRA --steps 4 --warmup 2 --no-e2e --no-cpu > gpurun_out/launches_${TAG}_${WL}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"monitor_kernel_(tma|masked|mma)" -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_${WL} -f \
    python bench.py --workload $WL $EXTRA --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/prof_${TAG}_${WL}.log 2>&1
