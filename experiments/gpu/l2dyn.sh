# C4 L2 eviction hints re-tested under the dynamic scheduler (C4 is now near DRAM-bound at 1.5x traffic);
# and which parity test the 16-date-stage build fails
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
D=paper_1807_01751_b200/libbwm.so; X=experiments/libs
BWM_LIB=$X/libbwm_r16s3.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | grep -E "FAILED|Error|assert" | head -8
for l in $X/libbwm_h2k5.so $X/libbwm_h1.so; do BWM_LIB=$l timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "lag or c4" 2>&1 | tail -1 | sed "s|^|$l parity: |"; done
ROUNDS=3 WL=C4 STEPS=20 bash experiments/ab_libs.sh $D $X/libbwm_h2k5.so $X/libbwm_h2k10.so $X/libbwm_h1.so 2>&1 | tee gpurun_out/l2dyn_C4.txt
