mkdir -p gpurun_out
TS_PROF=1 DENSE_ONLY_MASS=1 timeout 600 python tools/dense_bench.py tf32 1024 100 100 2>&1 | tail -4
TS_PROF=1 DENSE_NO_MASS=1 timeout 600 python tools/dense_bench.py tf32 1024 100 100 2>&1 | tail -4
