#!/bin/bash
# Interleaved bench A/B of libbwm builds (no parity step): ROUNDS rounds of A B C ...
WL=${WL:-C2}
ROUNDS=${ROUNDS:-3}
for r in $(seq $ROUNDS); do
  for lib in "$@"; do
    BWM_LIB=$lib timeout 200 python bench.py --workload $WL --nan-mode ${NANMODE:-fill} --no-e2e --no-cpu --steps ${STEPS:-40} --warmup 5 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
