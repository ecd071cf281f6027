# TALL (16-date stage) LEAN variant + L2 hints default: GPU suite, A/B BWM_TALL at C2, C4/C5 sanity
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/tall_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/tall_gputest.log; grep -E "FAILED|SKIPPED" gpurun_out/tall_gputest.log | head -12
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_env.sh BWM_TALL=1 BWM_TALL=0 2>&1 | tee gpurun_out/tall_C2.txt
ROUNDS=1 WL=C5 STEPS=10 bash experiments/ab_env.sh - 2>&1 | tee gpurun_out/tall_C5.txt
ROUNDS=2 WL=C4 STEPS=20 bash experiments/ab_env.sh - 2>&1 | tee gpurun_out/tall_C4.txt
