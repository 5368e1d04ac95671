set -x
export PYTHONUNBUFFERED=1
bash scripts/ab_lib_env.sh c2 30 "paper_1105_4002_b200/libtvreg_r1.so" "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg_u2.so" "paper_1105_4002_b200/libtvreg.so" > gpurun_out/ab_c2.log 2>&1
bash scripts/ab_lib_env.sh c5 10 "paper_1105_4002_b200/libtvreg_r1.so" "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_ILV=16" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_ILV=1" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_ZORDER=0" > gpurun_out/ab_c5.log 2>&1
bash scripts/ab_lib_env.sh c3 10 "paper_1105_4002_b200/libtvreg_r1.so" "paper_1105_4002_b200/libtvreg.so" > gpurun_out/ab_c3.log 2>&1
cat gpurun_out/ab_*.log
