# final round-2 validation at HEAD: GPU suite, smoke, default bench (+ C4/C5/mask/reference/n2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=r02end bash experiments/gpu/r2_val.sh
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" -c 400 --csv \
    --log-file gpurun_out/launches_r02end_C2.csv python bench.py --steps 4 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1; echo "launches rc=$?"
