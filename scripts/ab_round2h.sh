export PYTHONUNBUFFERED=1
bash scripts/ab_lib_env.sh c2 30 "paper_1105_4002_b200/libtvreg_base.so" "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg_base.so" "paper_1105_4002_b200/libtvreg.so" > gpurun_out/ab_search_c2.log 2>&1
grep -h " c2 " gpurun_out/ab_search_c2.log
python scripts/c4_study.py --only upn --out gpurun_out/c4_256h.json > gpurun_out/c4_256h.log 2>&1; cut -c1-260 gpurun_out/c4_256h.log
python scripts/upn_probe.py c2 > gpurun_out/upn_probe_h.log 2>&1; tail -n 1 gpurun_out/upn_probe_h.log | cut -c1-300
TVR_BENCH_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --steps 5 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; echo "dist1 rc=$?"; tail -c 1500 gpurun_out/bench_dist1.json; tail -n 5 gpurun_out/bench_dist1.err
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2h.log 2>&1; tail -n 3 gpurun_out/pytest_r2h.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2h.json 2> gpurun_out/bench_r2h.err; tail -c 300 gpurun_out/bench_r2h.json
