TS_ICVT=0 timeout 300 python tools/prof_eval.py fp64 30 8000000 255 20191223 > gpurun_out/ic.log 2>&1
TS_ICVT=1 timeout 300 python tools/prof_eval.py fp64 30 8000000 255 20191223 >> gpurun_out/ic.log 2>&1
TS_ICVT=1 timeout 600 python -m pytest tests -m gpu -q -x -k "wide or row_shard" > gpurun_out/t54.log 2>&1
