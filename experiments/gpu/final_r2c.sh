# last check at HEAD: GPU suite, smoke, default bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02h2}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -1 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C2.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_C4.log 2>&1
for f in gpurun_out/${TAG}_bench_*.log; do grep '^{' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d.get('roofline',{}); print(d['config'].get('workload','')[:30], 'ms', round(d['ms_per_step'],3), 'frac', r.get('frac'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'), 'e2e', (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('kind'), 'launches', d.get('gpu_launches'))"; done
