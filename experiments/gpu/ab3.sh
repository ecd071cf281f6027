# C4 occupancy variants (lagging cursor with smem tables), interleaved A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=experiments/libs
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_w12.so $L/libbwm_w16.so $L/libbwm_w8s3.so $L/libbwm_w12h.so $L/libbwm_hint1.so
