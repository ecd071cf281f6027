# monitoring-period fill on raw values (no centring per date): full GPU suite, then interleaved
# A/B against the previous build at C2, C4, C5
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/rawfill_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rawfill_tests.log
for wl in C2 C4 C5; do
  WL=$wl ROUNDS=3 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_old.so
done
