#!/bin/bash
# Interleaved A/B over environment settings: each argument is "NAME=VALUE ..." (or "-" for none)
WL=${WL:-C2}
ROUNDS=${ROUNDS:-3}
for r in $(seq $ROUNDS); do
  for envs in "$@"; do
    e=$envs; [ "$e" = "-" ] && e=""
    env $e timeout 200 python bench.py --workload $WL --nan-mode ${NANMODE:-fill} --no-e2e --no-cpu --steps 40 --warmup 5 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('[$envs]', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
