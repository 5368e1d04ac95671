export PYTHONUNBUFFERED=1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; tail -c 200 gpurun_out/bench_r2e.json
mkdir -p /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:spmv32s_kernel -s 2 -c 2 -o /tmp/ncu/c5 python scripts/profile_c5.py 3 > gpurun_out/ncu_c5_r2e.log 2>&1
ncu -i /tmp/ncu/c5.ncu-rep --page raw --csv > gpurun_out/c5_raw.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:"spmv16s|tv_kernel" -s 4 -c 4 -o /tmp/ncu/c3 python scripts/profile_step.py --config c3 --steps 3 > gpurun_out/ncu_c3_r2e.log 2>&1
ncu -i /tmp/ncu/c3.ncu-rep --page raw --csv > gpurun_out/c3_raw.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:"spmv16s|tv_kernel" -s 3 -c 3 -o /tmp/ncu/c2 python scripts/profile_step.py --config c2 --steps 3 > gpurun_out/ncu_c2_r2e.log 2>&1
ncu -i /tmp/ncu/c2.ncu-rep --page raw --csv > gpurun_out/c2_raw.csv 2>/dev/null
ncu -i /tmp/ncu/c2.ncu-rep --page source --csv --kernel-name regex:tv_kernel > gpurun_out/c2_tv_source.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2e.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/ncu_launch_r2e.log 2>&1
ls -la gpurun_out/*.csv; du -sh gpurun_out
