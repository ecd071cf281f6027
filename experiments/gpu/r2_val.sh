# round-2 validation: GPU suite, smoke, default bench line, C4/C5/mask lines, reference arm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02v}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C2.log 2>&1; echo "bench rc=$?"
for w in C4 C5; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_$w.log 2>&1; echo "bench $w rc=$?"; done
timeout 900 python bench.py --nan-mode mask --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_C2mask.log 2>&1; echo "bench mask rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --gpus 2 --pixels 16777216 --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_n2.log 2>&1; echo "n2 rc=$?"
for f in gpurun_out/${TAG}_bench_*.log; do echo "== $f"; grep '^{' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d.get('roofline',{}); print(d.get('impl','gpu'), d['n_gpus'], d['config'].get('workload','')[:40], 'ms', round(d['ms_per_step'],3), 'val', round(d['value'],2), 'frac', r.get('frac'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'), 'e2e', (d.get('e2e') or {}).get('value'), 'tp', r.get('tensor_pipe'))"; done
