# timing ablation: the TMA stage pipeline without the arithmetic (BWM_TMA_ABL=1, results wrong)
# vs the full kernel, C2/C4/C5
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in C2 C5 C4; do
  WL=$wl ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_abl.so
done
