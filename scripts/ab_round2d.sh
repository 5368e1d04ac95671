export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2d.log 2>&1; tail -n 3 gpurun_out/pytest_r2d.log
bash scripts/ab_lib_env.sh c5 10 "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_BLOCK=512" > gpurun_out/ab_c5d.log 2>&1
bash scripts/ab_lib_env.sh c2 30 "paper_1105_4002_b200/libtvreg.so" > gpurun_out/ab_c2d.log 2>&1
grep -h " c5 \| c2 " gpurun_out/ab_c5d.log gpurun_out/ab_c2d.log
python scripts/upn_probe.py c2 > gpurun_out/upn_probe_d.log 2>&1; tail -n 1 gpurun_out/upn_probe_d.log | cut -c1-400
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; tail -c 300 gpurun_out/bench_r2d.json
ncu --set full --clock-control none --import-source on -k regex:spmv32s_kernel -s 2 -c 2 -o gpurun_out/c5_r2d python scripts/profile_c5.py 3 > gpurun_out/ncu_c5_r2d.log 2>&1; tail -n 2 gpurun_out/ncu_c5_r2d.log
ncu --set full --clock-control none --import-source on -k regex:"spmv16s|tv_kernel" -s 4 -c 4 -o gpurun_out/c3_r2d python scripts/profile_step.py --config c3 --steps 3 > gpurun_out/ncu_c3_r2d.log 2>&1; tail -n 2 gpurun_out/ncu_c3_r2d.log
ncu --set full --clock-control none --import-source on -k regex:"spmv16s|tv_kernel" -s 3 -c 3 -o gpurun_out/c2_r2d python scripts/profile_step.py --config c2 --steps 3 > gpurun_out/ncu_c2_r2d.log 2>&1; tail -n 2 gpurun_out/ncu_c2_r2d.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2d.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/ncu_launch_r2d.log 2>&1; tail -n 2 gpurun_out/ncu_launch_r2d.log
