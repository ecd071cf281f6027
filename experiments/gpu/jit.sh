# just-in-time slice claims for long slices (C4) vs one-ahead pre-claims
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
ROUNDS=3 WL=C4 STEPS=20 bash experiments/ab_env.sh - BWM_SCHED_JIT=0 2>&1 | tee gpurun_out/jit_C4.txt
ROUNDS=2 WL=C5 STEPS=10 bash experiments/ab_env.sh - BWM_SCHED_JIT=1 2>&1 | tee gpurun_out/jit_C5.txt
ROUNDS=2 WL=C2 STEPS=40 bash experiments/ab_env.sh - BWM_SCHED_JIT=1 2>&1 | tee gpurun_out/jit_C2.txt
