# final evidence part B: masked captures + bench lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02f}
timeout 900 bash profiles/run_ncu.sh ${TAG}m C2 "--nan-mode mask"; echo "ncu C2 mask rc=$?"
timeout 900 bash profiles/run_ncu.sh ${TAG}m C4 "--nan-mode mask"; echo "ncu C4 mask rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C2.log 2>&1; echo "bench rc=$?"
for w in C4 C5; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_$w.log 2>&1; done
timeout 900 python bench.py --nan-mode mask --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_C2mask.log 2>&1
timeout 900 python bench.py --workload C4 --nan-mode mask --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_C4mask.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
du -sh gpurun_out
