TS_PROF=1 timeout 300 python tools/dense_bench.py tf32 1024 20 10 > gpurun_out/d3.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t31.log 2>&1
