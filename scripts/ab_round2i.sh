export PYTHONUNBUFFERED=1
python scripts/c4_study.py --only upn --out gpurun_out/c4_256i.json > gpurun_out/c4_256i.log 2>&1; cut -c1-230 gpurun_out/c4_256i.log
python scripts/upn_probe.py c2 > gpurun_out/upn_probe_i.log 2>&1; tail -n 1 gpurun_out/upn_probe_i.log | cut -c1-300
python scripts/run_config.py c2 30 | cut -c1-400
TVR_TV_ZC=22 python scripts/run_config.py c2 30 | cut -c1-400
TVR_TV_ZC=32 python scripts/run_config.py c2 30 | cut -c1-400
python -m pytest tests/test_gpu_solvers.py -q -x > gpurun_out/pytest_r2i.log 2>&1; tail -n 3 gpurun_out/pytest_r2i.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err; tail -c 300 gpurun_out/bench_r2i.json
