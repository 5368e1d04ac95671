export PYTHONUNBUFFERED=1
bash scripts/ab_env.sh c2 400 "TVR_SELL_MK_BLKCOST=2" "TVR_SELL_MK_BLKCOST=4" "TVR_SELL_MK_BLKCOST=6" "TVR_SELL_MK_BLKCOST=2" "TVR_SELL_MK_BLKCOST=4" 2>&1 | tee gpurun_out/ab_mk_blkcost.log
RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29511 TVR_BENCH_DIST=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; echo dist1 rc=$?; tail -c 400 gpurun_out/bench_dist1.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2m.csv python bench.py --steps 20 --warmup 5 > gpurun_out/ncu_launch_r2m.log 2>&1; tail -n 2 gpurun_out/ncu_launch_r2m.log | cut -c1-300
