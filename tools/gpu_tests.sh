mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo tests=$?; tail -4 gpurun_out/tall.log
grep -E "^FAILED|^E  " gpurun_out/tall.log | head -30
timeout 300 python bench.py --config eight_schools --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | tail -c 300
timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -1
