# validation at HEAD with the dynamic scheduler: GPU suite, smoke, bench lines, launch lists + ncu captures
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02d}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C2.log 2>&1; echo "bench rc=$?"
for w in C4 C5; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_$w.log 2>&1; done
for wl in C2 C4 C5; do timeout 900 bash profiles/run_ncu.sh $TAG $wl; echo "ncu $wl rc=$?"; done
for f in gpurun_out/${TAG}_bench_*.log; do echo "== $f"; grep '^{' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d.get('roofline',{}); print(d.get('impl','gpu'), d['config'].get('workload','')[:30], 'ms', round(d['ms_per_step'],3), 'val', round(d['value'],2), 'frac', r.get('frac'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'), 'e2e', (d.get('e2e') or {}).get('value'))"; done
du -sh gpurun_out
