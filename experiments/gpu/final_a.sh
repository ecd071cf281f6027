# final evidence part A: launch lists + ncu full captures of the fill kernels (C2, C4, C5)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02f}
for wl in C2 C4 C5; do timeout 900 bash profiles/run_ncu.sh $TAG $wl; echo "ncu $wl rc=$?"; done
du -sh gpurun_out
