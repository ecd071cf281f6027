# C4 (TMEM-parked 16-warp kernel, now closer to DRAM-bound): L2 eviction-priority hints again
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=experiments/libs
WL=C4 ROUNDS=3 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_h1.so $L/libbwm_h2.so $L/libbwm_h2f5.so
