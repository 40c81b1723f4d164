mkdir -p gpurun_out
timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -1
TS_PROF=1 timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | grep -v "pass ns by CTA" | tail -6
