# named CTA barrier every K stages (BWM_SYNC_EVERY=K) on the window-sum kernel: parity subset,
# then interleaved A/B at C2/C5/C4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BWM_LIB=experiments/libs/libbwm_sync1.so timeout 600 python -m pytest tests/test_gpu_parity.py -k "variants or shard or golden_parity_device or ragged" -x -q -p no:cacheprovider 2>&1 | tail -1
for wl in C2 C5; do
  WL=$wl ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_sync1.so experiments/libs/libbwm_sync2.so experiments/libs/libbwm_sync4.so experiments/libs/libbwm_sync8.so
done
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_sync1.so experiments/libs/libbwm_sync4.so
