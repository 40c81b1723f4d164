timeout 300 python tools/prof_eval.py fp64 200 > gpurun_out/w9.log 2>&1
timeout 300 python tools/prof_eval.py fp32 200 >> gpurun_out/w9.log 2>&1
TS_PROF=1 timeout 300 python tools/prof_run.py fp32 1000 1000 >> gpurun_out/w9.log 2>&1
TS_PROF=1 timeout 300 python tools/dense_bench.py tf32 1024 20 10 >> gpurun_out/w9.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t33.log 2>&1
