# quick check: fp64-policy parity tests + covtype pass / run timings per policy
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_covtype_fp32.py -q -x -k "logistic or covtype or tree or transition or run or ragged" -p no:cacheprovider > gpurun_out/tq.log 2>&1; echo tests=$?; tail -2 gpurun_out/tq.log
grep -E "^FAILED|^E  " gpurun_out/tq.log | head -10
for prec in fp64 fp32; do timeout 120 python tools/prof_eval.py $prec 200 | tail -1; done
for prec in fp64; do for i in 1 2; do timeout 300 python tools/prof_run.py $prec 200 200 2>&1 | tail -1; done; done
