# masked pass 3: crossing test per register block (lazy) instead of per date; masked GPU tests,
# then interleaved A/B against the previous build at C2 and C4 (mask)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_masked.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -k "mask" -m gpu -x -q -p no:cacheprovider > gpurun_out/lazy_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/lazy_tests.log
for wl in C2 C4; do
  NANMODE=mask STEPS=20 WL=$wl ROUNDS=3 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_old.so
done
