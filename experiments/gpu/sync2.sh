# named CTA barrier without a memory clobber (pacing only), K = 1, 4; A/B at C2/C5
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in C2 C5; do
  WL=$wl ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_sync1.so experiments/libs/libbwm_sync4.so
done
