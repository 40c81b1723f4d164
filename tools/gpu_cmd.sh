timeout 600 python -m pytest tests -m gpu -q -x -k "dense or tcgen05" > gpurun_out/t52.log 2>&1
for i in 1 2 3 4 5 6; do TS_PROF=1 timeout 60 python tools/dense_bench.py tf32 1024 20 10 >> gpurun_out/d13.log 2>&1; echo "iter $i rc=$?" >> gpurun_out/d13.log; done
