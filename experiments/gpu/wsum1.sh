# window-sum formulation: full GPU suite + C2/C4/C5 bench lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-ws1}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -30 gpurun_out/${TAG}_gputest.log | grep -v "^\s*$" | tail -25
for w in C2 C4 C5 C2 C4; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu > gpurun_out/${TAG}_$w.log 2>&1
  python - $w $TAG <<'PY'
import json,sys
for l in open(f"gpurun_out/{sys.argv[2]}_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]; print(sys.argv[1], "ms", round(d["ms_per_step"],3), "kernel", round(r["kernel_ms"],3), "frac", round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], r["launch"]["ring_mode"], r["launch"].get("ctas_per_sm_tma_lean"))
PY
done
