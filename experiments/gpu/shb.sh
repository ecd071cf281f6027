# CTA-shared 256-px (or 512-px) stage boxes re-measured on the window-sum kernel: parity subset,
# then interleaved A/B at C2/C5
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in experiments/libs/libbwm_shb.so experiments/libs/libbwm_shb6.so experiments/libs/libbwm_shb8w.so; do
  BWM_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py -k "variants or shard or golden_parity_device" -x -q -p no:cacheprovider 2>&1 | tail -1
done
for wl in C2 C5; do
  WL=$wl ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_shb.so experiments/libs/libbwm_shb6.so experiments/libs/libbwm_shb8w.so
done
