make -C paper_1912_11554_b200/csrc > gpurun_out/make.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t.log 2>&1; echo tests=$?
tail -3 gpurun_out/t.log
TS_PROF=1 timeout 120 python tools/prof_small.py gauss10
for m in thread warp; do timeout 300 python bench.py --config eight_schools --steps 2 --warmup 1 --no-cpu --exec-mode $m; done
for m in warp block; do timeout 300 python bench.py --config gauss10 --steps 3 --warmup 3 --no-cpu --exec-mode $m; done
