timeout 300 python tools/prof_eval.py fp64 200 > gpurun_out/w10.log 2>&1
for ns in 2 3 4; do TS_NSTAGE=$ns timeout 300 python tools/prof_run.py fp32 1000 1000 >> gpurun_out/w10.log 2>&1; done
timeout 300 python tools/prof_run.py fp64 1000 1000 >> gpurun_out/w10.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "logistic or covtype or tree or transition" > gpurun_out/t36.log 2>&1
