#!/bin/bash
# Time several builds of libtvreg on the same box: scripts/ab_multi.sh <config> <steps> <lib>...
CFG=$1; STEPS=$2; shift 2
for L in "$@"; do
  for rep in 1 2; do
    TVR_LIB_PATH=$PWD/$L timeout 300 python scripts/run_config.py $CFG $STEPS | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$L', d['config'], round(d['evals_per_s'],1), {k: round(d[k]['ms']*1000,1) for k in ('spmv_A','spmv_AT','tv_grad') if k in d})"
  done
done
