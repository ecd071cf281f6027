# quick A/B + parity: bench C2 (x2), C5, C4 and the fill-mode GPU parity suites
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_integration.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
for w in C2 C5 C4 C2; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu > gpurun_out/${TAG}_$w.log 2>&1
  python - $w <<'PY'
import json,sys
for l in open(f"gpurun_out/{__import__('os').environ.get('TAG','q')}_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]; print(sys.argv[1], "ms", round(d["ms_per_step"],3), "kernel", round(r["kernel_ms"],3), "frac", round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
