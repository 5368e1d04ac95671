export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2g.log 2>&1; tail -n 3 gpurun_out/pytest_r2g.log
python scripts/upn_probe.py c2 > gpurun_out/upn_probe_g.log 2>&1; tail -n 1 gpurun_out/upn_probe_g.log | cut -c1-300
python scripts/c4_study.py --only upn --out gpurun_out/c4_256g.json > gpurun_out/c4_256g.log 2>&1; cut -c1-300 gpurun_out/c4_256g.log
python scripts/c4_study.py --grid 32 --out gpurun_out/c4_32g.json > gpurun_out/c4_32g.log 2>&1; cut -c1-200 gpurun_out/c4_32g.log
python scripts/c4_study.py --only gpbb --out gpurun_out/c4_256g_gpbb.json > gpurun_out/c4_256g_gpbb.log 2>&1; cut -c1-300 gpurun_out/c4_256g_gpbb.log
