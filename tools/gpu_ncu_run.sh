mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_block_op --launch-skip 1 -c 1 -o gpurun_out/run_traj -f python tools/prof_run.py fp32 60 40 > gpurun_out/ncu_run.log 2>&1; echo ncu=$?
