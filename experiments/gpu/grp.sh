# 8-row groups for the ring loads/stores and the crossing search (no spills in the TALL kernels): parity + A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
P=experiments/libs/libbwm_prev.so; D=paper_1807_01751_b200/libbwm.so
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_libs.sh $D $P 2>&1 | tee gpurun_out/grp_C2.txt
ROUNDS=3 WL=C5 STEPS=10 bash experiments/ab_libs.sh $D $P 2>&1 | tee gpurun_out/grp_C5.txt
