# tensor-core fitted-value variant (BWM_MMA=1) vs the default at C4 (A/B + ncu), C5 ncu capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02m}
WL=C4 ROUNDS=2 bash experiments/ab_env.sh "-" "BWM_MMA=1"
BWM_MMA=1 timeout 900 bash profiles/run_ncu.sh ${TAG}mma C4; echo "ncu mma rc=$?"
timeout 900 bash profiles/run_ncu.sh $TAG C5; echo "ncu C5 rc=$?"
