#!/bin/bash
# scripts/ab_lib_env.sh <config> <steps> "<lib> <ENV=..> ..." ...   (each arg: a lib path then env settings)
CFG=$1; STEPS=$2; shift 2
for SPEC in "$@"; do
  set -- $SPEC; L=$1; shift
  env TVR_LIB_PATH=$PWD/$L "$@" timeout 300 python scripts/run_config.py $CFG $STEPS | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$SPEC'.replace('paper_1105_4002_b200/',''), d['config'], round(d['evals_per_s'],1), {k: round(d[k]['ms']*1000,1) for k in ('spmv_A','spmv_AT','tv_grad') if k in d})"
done
