# 16-warp lagging-cursor CTAs + device null draws: full GPU suite, C4 A/B (L2 hints), C4 ncu, lambda timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-w16}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/${TAG}_gputest.log
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_w16h.so
timeout 600 python experiments/crit_timing.py > gpurun_out/${TAG}_crit.log 2>&1; echo "crit rc=$?"; tail -8 gpurun_out/${TAG}_crit.log
timeout 900 bash profiles/run_ncu.sh $TAG C4; echo "ncu C4 rc=$?"
