# C4: pass-1 compensation state parked in TMEM (no spills at 16 warps; 20 warps possible)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=experiments/libs
for lib in $L/libbwm_p16.so $L/libbwm_p20.so; do BWM_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu -k "not masked" 2>&1 | tail -1 | sed "s|^|$lib: |"; done
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_p16.so $L/libbwm_p20.so $L/libbwm_w20.so
