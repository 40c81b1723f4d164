timeout 900 python bench.py > gpurun_out/bench_r1a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_block_op -c 1 -o gpurun_out/run_fp32_r1c python tools/prof_run.py fp32 60 40 > gpurun_out/ncu_run_d.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_block_op -c 1 -o gpurun_out/run_fp64_r1c python tools/prof_run.py fp64 60 40 > gpurun_out/ncu_run_e.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 0 --num-warmup 20 --num-samples 10 --single-precision --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
