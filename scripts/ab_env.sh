#!/bin/bash
# Time one build under several environment settings: scripts/ab_env.sh <config> <steps> "<ENV=..>" ...
CFG=$1; STEPS=$2; shift 2
for E in "$@"; do
  for rep in 1 2; do
    env $E timeout 300 python scripts/run_config.py $CFG $STEPS | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$E', d['config'], round(d['evals_per_s'],1), {k: round(d[k]['ms']*1000,1) for k in ('spmv_A','spmv_AT','tv_grad') if k in d})"
  done
done
