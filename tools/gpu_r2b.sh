# profiling batch: new test, stage/L2 sweeps of the fp32 covtype pass, TS_PROF breakdown, ncu of the pass
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "adaptation_replay or runs_match" -p no:cacheprovider > gpurun_out/t_replay.log 2>&1; echo replay=$?; tail -3 gpurun_out/t_replay.log
for ns in 1 2 3 4; do for k in 0 70; do echo "NSTAGE=$ns KEEP=$k"; TS_NSTAGE=$ns TS_L2_KEEP=$k timeout 120 python tools/prof_eval.py fp32 200 | tail -1; done; done > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
TS_PROF=1 timeout 300 python tools/prof_run.py fp32 60 40 > gpurun_out/prof_run.log 2>&1; tail -12 gpurun_out/prof_run.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_block_op --launch-skip 1 -c 1 -o gpurun_out/eval_fp32 -f python tools/prof_eval.py fp32 20 > gpurun_out/ncu_eval.log 2>&1; echo ncu=$?
