cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cols in 256 512; do
  echo "== BWM_TMEM_COLS_MAX=$cols"
  BWM_TMEM_COLS_MAX=$cols timeout 600 python bench.py --workload C4 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/c4_cols$cols.log 2>&1
  python - <<PY
import json
for l in open("gpurun_out/c4_cols$cols.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]; print("cols=$cols", "ms", round(d["ms_per_step"],3), "frac", round(r["frac"],3), r["launch"]["ring_mode"], r["launch"]["ctas_per_sm_tma_lean"], d["clocks"])
PY
  tail -2 gpurun_out/c4_cols$cols.log | grep -v "^{" 
done
BWM_TMEM_COLS_MAX=512 timeout 900 python -m pytest tests/test_gpu_fullsize.py -k "C4" tests/test_gpu_parity.py -x -q > gpurun_out/c4_512_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c4_512_tests.log
