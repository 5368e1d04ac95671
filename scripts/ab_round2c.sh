export PYTHONUNBUFFERED=1
bash scripts/ab_lib_env.sh c2 30 "paper_1105_4002_b200/libtvreg_v0.so" "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg_v4.so" "paper_1105_4002_b200/libtvreg.so" > gpurun_out/ab_tv2_c2.log 2>&1
bash scripts/ab_lib_env.sh c3 10 "paper_1105_4002_b200/libtvreg_v0.so" "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg_v4.so" > gpurun_out/ab_tv2_c3.log 2>&1
grep -h " c2 \| c3 " gpurun_out/ab_tv2_c2.log gpurun_out/ab_tv2_c3.log
bash scripts/ab_lib_env.sh c5 10 "paper_1105_4002_b200/libtvreg.so" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_L2=1" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_L2=2" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_L2=3" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_L2=3 TVR_SELL32_ILV=16" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_UNROLL=3" "paper_1105_4002_b200/libtvreg.so TVR_SELL32_BLOCK=1024" > gpurun_out/ab_l2_c5.log 2>&1
grep -h " c5 " gpurun_out/ab_l2_c5.log
python scripts/upn_probe.py c2 > gpurun_out/upn_probe.log 2>&1
TVR_LIB_PATH=$PWD/paper_1105_4002_b200/libtvreg_r1.so python scripts/upn_probe.py c2 >> gpurun_out/upn_probe.log 2>&1
cat gpurun_out/upn_probe.log | tail -n 4
