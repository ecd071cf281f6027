# 16-date stages and 8-warp ring CTAs under the dynamic slice scheduler
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
D=paper_1807_01751_b200/libbwm.so; X=experiments/libs
for l in $X/libbwm_r16s3.so $X/libbwm_rw8.so; do BWM_LIB=$l timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1 | sed "s|^|$l parity: |"; done
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_libs.sh $D $X/libbwm_r16s3.so $X/libbwm_r16s2.so $X/libbwm_rw8.so 2>&1 | tee gpurun_out/tune2_C2.txt
ROUNDS=2 WL=C5 STEPS=10 bash experiments/ab_libs.sh $D $X/libbwm_r16s3.so $X/libbwm_r16s2.so $X/libbwm_rw8.so 2>&1 | tee gpurun_out/tune2_C5.txt
ROUNDS=2 WL=C4 STEPS=20 bash experiments/ab_libs.sh $D $X/libbwm_r16s3.so 2>&1 | tee gpurun_out/tune2_C4.txt
