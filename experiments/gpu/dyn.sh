# dynamic per-warp slice scheduler of the TMA kernel (BWM_DYN=1 default) vs the static schedule
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/dyn_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/dyn_gputest.log
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_env.sh BWM_DYN=1 BWM_DYN=0 2>&1 | tee gpurun_out/dyn_C2.txt
ROUNDS=3 WL=C5 STEPS=10 bash experiments/ab_env.sh BWM_DYN=1 BWM_DYN=0 2>&1 | tee gpurun_out/dyn_C5.txt
ROUNDS=3 WL=C4 STEPS=20 bash experiments/ab_env.sh BWM_DYN=1 BWM_DYN=0 2>&1 | tee gpurun_out/dyn_C4.txt
