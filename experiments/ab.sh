#!/bin/bash
# A/B of experimental libbwm builds: parity tests per variant, then interleaved bench runs
# (ROUNDS rounds of A B C ...), so clock / power-cap drift hits every variant alike.
WL=${WL:-C2}
ROUNDS=${ROUNDS:-2}
for lib in "$@"; do
  BWM_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_masked.py -x -q -m gpu 2>&1 | tail -1 | sed "s|^|$lib parity: |"
done
for r in $(seq $ROUNDS); do
  for lib in "$@"; do
    BWM_LIB=$lib timeout 200 python bench.py --workload $WL --nan-mode ${NANMODE:-fill} --no-e2e --no-cpu --steps 40 --warmup 5 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['roofline']['launch']['ctas_per_sm_tma'], d['roofline']['launch'].get('ctas_per_sm_tma_lean'), d['roofline']['launch']['tmem_cols'])"
  done
done
