mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -x -m gpu -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo tests=$?; tail -3 gpurun_out/tall.log
timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -2
timeout 300 python tools/prof_run.py fp64 100 100 2>&1 | tail -1
TS_PROF=1 timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | grep -v "pass ns by CTA" | tail -6
