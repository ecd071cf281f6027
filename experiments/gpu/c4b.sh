# sanitizer over the lagging-cursor kernels + C4 warps/stages A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -x -q -m gpu 2>&1 | tail -3
L=experiments/libs
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_w8s4.so $L/libbwm_w12s3.so $L/libbwm_w8s5.so
