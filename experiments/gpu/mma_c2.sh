# tensor-core fitted values at C2: the default (TMEM residual ring, FFMA2) vs the lagging cursor
# forced by a 64-column TMEM cap, on FFMA2 and on tcgen05.mma (BWM_MMA=1); parity of the MMA
# variant at full C2 size; ncu capture of the MMA variant for its tensor-pipe figures.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BWM_MMA=1 BWM_TMEM_COLS_MAX=64 timeout 900 python -m pytest tests/test_gpu_fullsize.py -k C2 -x -q > gpurun_out/mma_c2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/mma_c2_tests.log
WL=C2 ROUNDS=3 bash experiments/ab_env.sh "-" "BWM_TMEM_COLS_MAX=64" "BWM_TMEM_COLS_MAX=64 BWM_MMA=1"
BWM_MMA=1 BWM_TMEM_COLS_MAX=64 timeout 900 bash profiles/run_ncu.sh r02mma C2; echo "ncu mma rc=$?"
