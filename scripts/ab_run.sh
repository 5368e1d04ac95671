#!/bin/bash
# A/B: alternate the previous build (libtvreg_prev.so) and the current one on the same box.
# usage: scripts/ab_run.sh <config> <steps> <reps> [out]
CFG=${1:-c2}; STEPS=${2:-50}; REPS=${3:-2}; OUT=${4:-gpurun_out/ab.json}
mkdir -p gpurun_out; : > $OUT
for i in $(seq $REPS); do
  TVR_LIB_PATH=$PWD/paper_1105_4002_b200/libtvreg_prev.so timeout 300 python scripts/run_config.py $CFG $STEPS | sed 's/^{/{"build": "prev", /' >> $OUT
  timeout 300 python scripts/run_config.py $CFG $STEPS | sed 's/^{/{"build": "cur", /' >> $OUT
done
python - $OUT <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(d["build"], d["config"], round(d["evals_per_s"], 1), {k: round(d[k]["ms"], 4) for k in ("spmv_A", "spmv_AT", "tv_grad") if k in d})
PY
