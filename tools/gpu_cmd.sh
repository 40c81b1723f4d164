timeout 600 python -m pytest tests -m gpu -q -x -k "dense or tcgen05" > gpurun_out/t39.log 2>&1
TS_PROF=1 timeout 300 python tools/dense_bench.py tf32 1024 20 10 > gpurun_out/d5.log 2>&1
