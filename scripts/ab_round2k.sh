export PYTHONUNBUFFERED=1
mkdir -p gpurun_out /tmp/ncu
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2k.log 2>&1; tail -n 3 gpurun_out/pytest_r2k.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2k.json 2> gpurun_out/bench_r2k.err; tail -c 300 gpurun_out/bench_r2k.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2k.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/ncu_launch_r2k.log 2>&1; tail -n 2 gpurun_out/ncu_launch_r2k.log
ncu --set full --clock-control none --import-source on -k regex:"spmv16s|tv_row" -s 3 -c 3 -o /tmp/ncu/c2k python scripts/profile_step.py --config c2 --steps 3 > gpurun_out/ncu_c2_r2k.log 2>&1; tail -n 2 gpurun_out/ncu_c2_r2k.log
ncu -i /tmp/ncu/c2k.ncu-rep --page raw --csv > gpurun_out/c2_raw_r2k.csv 2>/dev/null
ls -la gpurun_out/c2_raw_r2k.csv
