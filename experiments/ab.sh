#!/bin/bash
# A/B of experimental libbwm builds: bench C2 (device-resident) per variant, parity tests per variant
for lib in "$@"; do
  for i in 1 2; do
    BWM_LIB=$lib timeout 200 python bench.py --no-e2e --no-cpu --steps 40 --warmup 5 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['roofline']['launch']['ctas_per_sm_tma'])"
  done
done
