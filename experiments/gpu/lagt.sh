# C4 lagging cursor (kRingLagT): warps per CTA x stages per warp (with the TMEM-parked
# compensation state), interleaved against the default 16 x 2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in experiments/libs/libbwm_w12s3.so experiments/libs/libbwm_w8s4.so; do
  BWM_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -k "c4_tile or lagging" -x -q -p no:cacheprovider 2>&1 | tail -1
done
WL=C4 ROUNDS=3 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_w12s3.so experiments/libs/libbwm_w8s4.so experiments/libs/libbwm_w16s2.so
