#!/bin/bash
# Sweep the CTA partition model of the sliced-ELL passes: per-CTA spread (sell_prof) and pass times.
CFG=${1:-c2}
for L in 0 25 50 75 100; do
  export TVR_SELL_MK_LAMBDA=$L
  python scripts/sell_prof.py $CFG 30 2>/dev/null | python -c "
import json,sys,numpy as np
d=json.loads(sys.stdin.read())
for k,v in d.items():
    a=np.array(v['mean_dur_by_cta_us'])
    print('lambda $L',k,'mean',a.mean().round(1),'min',a.min(),'max',a.max(),'median span',sorted(v['span_us'])[len(v['span_us'])//2])"
  python scripts/run_config.py $CFG 300 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('lambda $L', round(d['evals_per_s'],1), {k: round(d[k]['ms']*1000,1) for k in ('spmv_A','spmv_AT','tv_grad') if k in d})"
done
