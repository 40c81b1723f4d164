mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -x -m gpu -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo tests=$?; tail -3 gpurun_out/tall.log
grep -E "dense tf32 decision replay" -A0 gpurun_out/tall.log | cut -c1-300
timeout 300 python tools/prof_eval.py fp64x 100 | tail -1
timeout 300 python tools/prof_run.py fp64x 60 40 2>&1 | tail -1
DENSE_ONLY_MASS=1 timeout 600 python tools/dense_bench.py tf32 1024 100 100 2>&1 | tail -2
