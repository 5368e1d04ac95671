# round 2: GPU tests, stencil A/B, default bench, c5 A-pass capture
export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_r2c.log 2>&1
tail -n 5 gpurun_out/pytest_r2c.log
bash scripts/ab_lib_env.sh c2 30 "paper_1105_4002_b200/libtvreg_v0.so" "paper_1105_4002_b200/libtvreg_v1.so" "paper_1105_4002_b200/libtvreg_v2.so" "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg_v0.so" > gpurun_out/ab_tv_c2.log 2>&1
bash scripts/ab_lib_env.sh c3 10 "paper_1105_4002_b200/libtvreg_v0.so" "paper_1105_4002_b200/libtvreg_v1.so" "paper_1105_4002_b200/libtvreg_v2.so" "paper_1105_4002_b200/libtvreg.so" > gpurun_out/ab_tv_c3.log 2>&1
grep -h "c2\|c3" gpurun_out/ab_tv_c2.log gpurun_out/ab_tv_c3.log | grep -v Trace
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
tail -c 600 gpurun_out/bench_r2c.json
ncu --set full --clock-control none --import-source on -k regex:spmv32s_kernel -s 2 -c 1 -o gpurun_out/c5_A_r2 python scripts/profile_c5.py 3 > gpurun_out/ncu_c5_r2.log 2>&1
tail -n 3 gpurun_out/ncu_c5_r2.log
