timeout 600 python -m pytest tests -m gpu -q -x -k "dense or tcgen05" > gpurun_out/t56.log 2>&1
for i in 1 2; do TS_PROF=1 timeout 120 python tools/dense_bench.py tf32 1024 20 10 >> gpurun_out/d14.log 2>&1; echo "rc=$?" >> gpurun_out/d14.log; done
