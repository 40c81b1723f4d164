for i in $(seq 1 14); do timeout 60 python tools/dense_bench.py tf32 1024 20 10 > gpurun_out/d9_$i.log 2>&1; echo "iter $i rc=$?" >> gpurun_out/d9.log; done
timeout 600 python -m pytest tests -m gpu -q -x -k "dense or tcgen05" > gpurun_out/t42.log 2>&1
