mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" -p no:cacheprovider 2>&1 | tail -2
TS_PROF=1 DENSE_ONLY_MASS=1 timeout 600 python tools/dense_bench.py tf32 1024 100 100 2>&1 | tail -3
DENSE_ONLY_MASS=1 timeout 600 python tools/dense_bench.py fp64 256 30 30 2>&1 | tail -1
