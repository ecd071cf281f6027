# masked LEAN variant (no MOSUM mean accumulation unless requested); tests + A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_masked.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -2
WL=C2 NANMODE=mask ROUNDS=2 STEPS=10 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_m7.so
