mkdir -p gpurun_out
run() { for c in eight_schools gauss10; do timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $c', d['value'])"; done; timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -1 | sed "s/^/$1 /"; }
run glibc
make -C paper_1912_11554_b200/csrc clean > /dev/null; make -C paper_1912_11554_b200/csrc -j16 EXTRA=-DTS_CUDA_LIBM > gpurun_out/mk.log 2>&1 || tail -5 gpurun_out/mk.log
run cuda
