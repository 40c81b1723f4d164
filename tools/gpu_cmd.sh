for v in 0 1 2; do TS_ICVT=$v timeout 300 python tools/prof_eval.py fp64 30 8000000 255 20191223 >> gpurun_out/ic2.log 2>&1; done
TS_ICVT=2 timeout 600 python -m pytest tests -m gpu -q -x -k "wide or row_shard" > gpurun_out/t55.log 2>&1
