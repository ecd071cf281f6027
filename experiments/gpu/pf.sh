# L2 tensor prefetch of the CTA tile's rows (BWM_TMA_PF distance, _ALL: every warp vs round robin)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L="experiments/libs/libbwm_pf4_0.so experiments/libs/libbwm_pf8_0.so experiments/libs/libbwm_pf4_1.so experiments/libs/libbwm_pf12_0.so"
BWM_LIB=experiments/libs/libbwm_pf8_0.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L 2>&1 | tee gpurun_out/pf_C2.txt
ROUNDS=2 WL=C5 STEPS=10 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L 2>&1 | tee gpurun_out/pf_C5.txt
ROUNDS=2 WL=C4 STEPS=20 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L 2>&1 | tee gpurun_out/pf_C4.txt
