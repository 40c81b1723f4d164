make -C paper_1912_11554_b200/csrc > gpurun_out/make.log 2>&1 || exit 1
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/t.log 2>&1; echo tests=$?
tail -3 gpurun_out/t.log
for m in warp block; do timeout 300 python bench.py --config gauss10 --steps 3 --warmup 3 --no-cpu --exec-mode $m; done
timeout 300 python bench.py --config eight_schools --steps 2 --warmup 1 --no-cpu --exec-mode thread
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e
