for r in 1 4 8; do TS_NREP=$r TS_PROF=1 timeout 300 python tools/prof_run.py fp32 1000 1000 >> gpurun_out/w12.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "logistic or wide or row_shard or covtype" > gpurun_out/t38.log 2>&1
