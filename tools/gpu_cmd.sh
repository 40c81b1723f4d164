timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t27.log 2>&1
timeout 900 python bench.py --config rowshard --steps 2 --warmup 1 --num-warmup 100 --num-samples 100 > gpurun_out/b6.log 2>&1
timeout 900 python bench.py --config rowshard --precision fp64 --steps 1 --warmup 1 --num-warmup 30 --num-samples 30 >> gpurun_out/b6.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_block_op -c 1 -o gpurun_out/wide_fp64 python tools/prof_eval.py fp64 5 8000000 255 20191223 > gpurun_out/ncu_wide4.log 2>&1
