# TMA tensor-map L2 promotion (BWM_L2PROMO 0 none / 1 64B / 2 128B / 3 256B, the default)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_env.sh BWM_L2PROMO=3 BWM_L2PROMO=0 BWM_L2PROMO=1 BWM_L2PROMO=2 2>&1 | tee gpurun_out/promo_C2.txt
ROUNDS=2 WL=C5 STEPS=10 bash experiments/ab_env.sh BWM_L2PROMO=3 BWM_L2PROMO=0 BWM_L2PROMO=2 2>&1 | tee gpurun_out/promo_C5.txt
ROUNDS=2 WL=C4 STEPS=20 bash experiments/ab_env.sh BWM_L2PROMO=3 BWM_L2PROMO=0 BWM_L2PROMO=2 2>&1 | tee gpurun_out/promo_C4.txt
