# masked C4 (global rings): 3-stage x x^T ring frees shared memory for L1 (the rings live there)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BWM_LIB=experiments/libs/libbwm_bs3.so timeout 900 python -m pytest tests/test_masked.py tests/test_gpu_fuzz.py -x -q -m gpu -k "mask" 2>&1 | tail -1
WL=C4 NANMODE=mask ROUNDS=2 STEPS=4 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_bs3.so
