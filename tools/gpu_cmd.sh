timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t47.log 2>&1
for i in 1 2; do TS_PROF=1 timeout 120 python tools/dense_bench.py tf32 1024 20 10 >> gpurun_out/d12.log 2>&1; echo "rc=$?" >> gpurun_out/d12.log; done
timeout 300 python tools/prof_run.py fp32 1000 1000 >> gpurun_out/d12.log 2>&1
