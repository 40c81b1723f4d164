timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t18.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 15 > gpurun_out/bench4.log 2>&1
timeout 600 python bench.py --config eight_schools --steps 2 --warmup 1 >> gpurun_out/bench4.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 >> gpurun_out/bench4.log 2>&1
