# TALL stages without ring mirror rows where mirrors would not fit (C5): parity + A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
ROUNDS=3 WL=C5 STEPS=10 bash experiments/ab_env.sh BWM_TALL_NOMIRROR=1 BWM_TALL_NOMIRROR=0 2>&1 | tee gpurun_out/tallnm_C5.txt
ROUNDS=2 WL=C2 STEPS=40 bash experiments/ab_env.sh - 2>&1 | tee gpurun_out/tallnm_C2.txt
