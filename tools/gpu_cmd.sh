timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t58.log 2>&1
TS_PROF=1 timeout 300 python tools/prof_run.py fp32 1000 1000 > gpurun_out/th.log 2>&1
RUN_SEED=1001 TS_PROF=1 timeout 300 python tools/prof_run.py fp32 1000 1000 >> gpurun_out/th.log 2>&1
