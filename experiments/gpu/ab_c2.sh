# C2/C4 A/B: two-chain S-dot (default) vs one chain; C2 stage shapes (8- vs 16-date stages, ring depth)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=experiments/libs
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -2
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_chain1.so
WL=C2 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_chain1.so $L/libbwm_s4.so $L/libbwm_s6.so $L/libbwm_r16s3.so $L/libbwm_r16s4.so
