timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t49.log 2>&1
RUN_SEED=1001 TS_PROF=1 timeout 300 python tools/prof_run.py fp32 1000 1000 > gpurun_out/ps5.log 2>&1
timeout 600 python bench.py --config eight_schools --steps 3 --warmup 3 >> gpurun_out/ps5.log 2>&1
timeout 300 python tools/single_chain.py >> gpurun_out/ps5.log 2>&1
