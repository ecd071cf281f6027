cd $GRAFT_REPO_ROOT
python experiments/gpu/fz.py
timeout 1500 python -m pytest tests/test_masked.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
WL=C2 NANMODE=mask ROUNDS=2 STEPS=10 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_m5.so
WL=C4 NANMODE=mask ROUNDS=1 STEPS=4 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_m5.so
