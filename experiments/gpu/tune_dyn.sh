# re-tune stage depth (TMEM ring) and C4 warps x stages with the dynamic slice scheduler
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
D=paper_1807_01751_b200/libbwm.so; X=experiments/libs
BWM_LIB=$X/libbwm_l12x3.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "lag or c4" 2>&1 | tail -1
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_libs.sh $D $X/libbwm_s4.so $X/libbwm_s6.so 2>&1 | tee gpurun_out/tune_C2.txt
ROUNDS=2 WL=C5 STEPS=10 bash experiments/ab_libs.sh $D $X/libbwm_s4.so $X/libbwm_s6.so 2>&1 | tee gpurun_out/tune_C5.txt
ROUNDS=3 WL=C4 STEPS=20 bash experiments/ab_libs.sh $D $X/libbwm_l12x3.so $X/libbwm_l8x4.so 2>&1 | tee gpurun_out/tune_C4.txt
