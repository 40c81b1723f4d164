mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "logistic or covtype or tree or run or transition or fp64x" -p no:cacheprovider > gpurun_out/tq.log 2>&1; echo tests=$?; tail -3 gpurun_out/tq.log
for ic in 0 1 2; do echo "ICVT=$ic"; TS_ICVT=$ic timeout 120 python tools/prof_eval.py fp64 200 | tail -1; done
timeout 120 python tools/prof_eval.py fp32 200 | tail -1
timeout 300 python tools/prof_run.py fp64 100 100 2>&1 | tail -1
timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_block_op --launch-skip 1 -c 1 -o gpurun_out/run_fp32 -f python tools/prof_run.py fp32 60 40 > gpurun_out/ncu_run.log 2>&1; echo ncu=$?
