#!/bin/bash
# A/B of experimental libbwm builds: bench C2 (device-resident) per variant + parity tests
WL=${WL:-C2}
for lib in "$@"; do
  BWM_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_masked.py -x -q -m gpu 2>&1 | tail -1 | sed "s|^|$lib parity: |"
  for i in 1 2; do
    BWM_LIB=$lib timeout 200 python bench.py --workload $WL --nan-mode ${NANMODE:-fill} --no-e2e --no-cpu --steps 40 --warmup 5 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['roofline']['launch']['ctas_per_sm_tma'], d['roofline']['launch'].get('ctas_per_sm_tma_lean'), d['roofline']['launch']['tmem_cols'])"
  done
done
