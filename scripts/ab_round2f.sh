export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2f.log 2>&1; tail -n 3 gpurun_out/pytest_r2f.log
python scripts/upn_probe.py c2 > gpurun_out/upn_probe_f.log 2>&1; tail -n 1 gpurun_out/upn_probe_f.log | cut -c1-600
TVR_EXT_EVAL=0 python scripts/upn_probe.py c2 >> gpurun_out/upn_probe_f.log 2>&1; tail -n 1 gpurun_out/upn_probe_f.log | cut -c1-600
python scripts/c4_study.py --grid 32 --out gpurun_out/c4_32f.json > gpurun_out/c4_32f.log 2>&1; cut -c1-250 gpurun_out/c4_32f.log
python scripts/c4_study.py --only upn --out gpurun_out/c4_256f.json > gpurun_out/c4_256f.log 2>&1; cut -c1-400 gpurun_out/c4_256f.log
