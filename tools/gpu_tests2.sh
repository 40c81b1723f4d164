mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo tests=$?; tail -3 gpurun_out/tall.log
grep -E "^FAILED|^E  " gpurun_out/tall.log | head -20
for c in eight_schools gauss10; do timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d.get('unit'))"; done
