# isolate the C4 mask slowdown: X staged + 3-stage B ring (default now), X staged + 4 stages (1 CTA/SM),
# X global (BWM_MASK_XG=1, 4 stages as round 1)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
WL=C4 NANMODE=mask ROUNDS=1 STEPS=4 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_xs4.so experiments/libs/libbwm_mx0.so
WL=C4 NANMODE=mask ROUNDS=1 STEPS=4 bash experiments/ab_env.sh "BWM_MASK_XG=1"
