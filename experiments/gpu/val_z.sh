# new masked/chunked test first, then the round-2 validation (GPU suite, smoke, bench lines)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_masked.py -m gpu -k chunked -x -q -p no:cacheprovider > gpurun_out/z_chunked.log 2>&1; echo "chunked rc=$?"; tail -3 gpurun_out/z_chunked.log
TAG=r02z bash experiments/gpu/r2_val.sh
