# masked-mode check: GPU tests, then short C2/C5/C4 timings (each bounded by timeout)
timeout 300 python -m pytest tests/test_masked.py -q -m gpu -x 2>&1 | tail -4
for wl in C2 C5 C4; do timeout 240 python bench.py --nan-mode mask --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],2), round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['launch'].get('ctas_per_sm_masked'))"; done
