export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2j.log 2>&1; tail -n 3 gpurun_out/pytest_r2j.log
for zc in 0 22 32; do TVR_TV_ZC=$zc python scripts/run_config.py c2 30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 zc=$zc', round(d['evals_per_s'],1), round(d['tv_grad']['ms']*1e3,2))"; done
for zc in 0 16 64; do TVR_TV_ZC=$zc python scripts/run_config.py c3 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 zc=$zc', round(d['evals_per_s'],1), round(d['tv_grad']['ms']*1e3,2))"; done
TVR_EXT_EVAL_AT=1 python scripts/upn_probe.py c2 > gpurun_out/upn_probe_j.log 2>&1; tail -n 1 gpurun_out/upn_probe_j.log | cut -c1-700
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2j.json 2> gpurun_out/bench_r2j.err; tail -c 200 gpurun_out/bench_r2j.json
