# round-2 final evidence: GPU suite + sanitizer, smoke, launch lists + ncu full captures (C2, C4, C5,
# C2 mask, C4 mask), bench lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02f}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
for wl in C2 C4 C5; do timeout 900 bash profiles/run_ncu.sh $TAG $wl; echo "ncu $wl rc=$?"; done
timeout 900 bash profiles/run_ncu.sh ${TAG}m C2 "--nan-mode mask"; echo "ncu C2 mask rc=$?"
timeout 900 bash profiles/run_ncu.sh ${TAG}m C4 "--nan-mode mask"; echo "ncu C4 mask rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C2.log 2>&1; echo "bench rc=$?"
for w in C4 C5; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_$w.log 2>&1; done
timeout 900 python bench.py --nan-mode mask --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_C2mask.log 2>&1
timeout 900 python bench.py --workload C4 --nan-mode mask --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_C4mask.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
for f in gpurun_out/${TAG}_bench_*.log; do echo "== $f"; grep '^{' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d.get('roofline',{}); print(d.get('impl','gpu'), d['config'].get('workload','')[:30], 'ms', round(d['ms_per_step'],3), 'val', round(d['value'],2), 'frac', r.get('frac'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'), 'e2e', (d.get('e2e') or {}).get('value'))"; done
