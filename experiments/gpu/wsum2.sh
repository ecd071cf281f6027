# window-sum formulation, round 2: full GPU suite, C4 A/B (L1 tables, L2 hints, 8-warp CTAs), ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-ws2}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/${TAG}_gputest.log
WL=C4 ROUNDS=2 bash experiments/ab_env.sh "-" "BWM_TMA_LAGL1=1"
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_hint1.so experiments/libs/libbwm_hint2.so experiments/libs/libbwm_w8.so
timeout 900 bash profiles/run_ncu.sh $TAG C4; echo "ncu C4 rc=$?"
timeout 900 bash profiles/run_ncu.sh $TAG C2; echo "ncu C2 rc=$?"
