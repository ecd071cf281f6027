
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_gputest.log 2>&1; echo "gputest rc=$?"
tail -5 gpurun_out/r2_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2_smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_c2.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/r2_bench_c2.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/r2_bench_ref.log
timeout 900 python bench.py --gpus 2 --pixels 16777216 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench_n2.log 2>&1; echo "n2 rc=$?"; tail -c 2500 gpurun_out/r2_bench_n2.log
