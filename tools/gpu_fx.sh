mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "logistic or covtype or row_shard or trajectory" -p no:cacheprovider 2>&1 | tail -2
for c in 1 2 4 8; do echo "copies=$c: $(TS_FX_COPIES=$c timeout 120 python tools/prof_eval.py fp32 300 | tail -1 | cut -c1-95)"; done
for c in 2 4 8; do for i in 1 2; do echo "copies=$c $(TS_FX_COPIES=$c timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -1 | cut -c30-110)"; done; done
