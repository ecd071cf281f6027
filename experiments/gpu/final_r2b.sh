# end-of-round evidence at HEAD (grouped ring access): GPU suite, smoke, bench lines, C2 ncu; A/B of 3 TALL stages
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r02g}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/${TAG}_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C2.log 2>&1; echo "bench rc=$?"
for w in C4 C5; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_$w.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
timeout 900 bash profiles/run_ncu.sh $TAG C2; echo "ncu C2 rc=$?"
ROUNDS=3 WL=C2 STEPS=40 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_ts3.so 2>&1 | tee gpurun_out/ts3_C2.txt
for f in gpurun_out/${TAG}_bench_*.log; do echo "== $f"; grep '^{' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); r=d.get('roofline',{}); print(d.get('impl','gpu'), d['config'].get('workload','')[:30], 'ms', round(d['ms_per_step'],3), 'val', round(d['value'],2), 'frac', r.get('frac'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'), 'e2e', (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('kind'))"; done
