mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo tests=$?; tail -3 gpurun_out/tall.log
grep -E "^FAILED|^E  " gpurun_out/tall.log | head -20
for c in eight_schools gauss10; do timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'])"; done
for i in 1 2; do timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -1; done
DENSE_ONLY_MASS=1 timeout 600 python tools/dense_bench.py tf32 1024 100 100 2>&1 | tail -1
