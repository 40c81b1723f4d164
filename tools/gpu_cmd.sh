timeout 300 python tools/prof_eval.py fp64 200 > gpurun_out/w11.log 2>&1
TS_PROF=1 timeout 300 python tools/dense_bench.py tf32 1024 20 10 >> gpurun_out/w11.log 2>&1
timeout 600 python bench.py --config eight_schools --steps 3 --warmup 3 >> gpurun_out/w11.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t37.log 2>&1
