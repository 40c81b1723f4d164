# quick check: logistic parity tests + eval-only pass timing + short run timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_covtype_fp32.py -q -x -k "logistic or covtype or tree or run or transition" -p no:cacheprovider > gpurun_out/tq.log 2>&1; echo tests=$?; tail -3 gpurun_out/tq.log
for prec in fp32 fp64; do timeout 120 python tools/prof_eval.py $prec 200 | tail -1; done
timeout 300 python tools/prof_run.py fp32 200 200 2>&1 | tail -2
TS_PROF=1 timeout 300 python tools/prof_run.py fp32 60 40 2>&1 | grep -v "pass ns by CTA" | tail -4
