# masked-kernel ablations (timing only, results wrong): where does the C2 mask time go?
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=experiments/libs
WL=C2 NANMODE=mask ROUNDS=2 STEPS=10 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_abl1.so $L/libbwm_abl2.so $L/libbwm_abl4.so $L/libbwm_abl8.so $L/libbwm_abl7.so
