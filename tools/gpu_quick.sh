# quick check: full GPU tests + covtype pass / run timings per policy
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo tests=$?; tail -2 gpurun_out/tall.log
grep -E "^FAILED|^E  " gpurun_out/tall.log | head -20
for prec in fp32 fp64 fp64x; do timeout 120 python tools/prof_eval.py $prec 200 | tail -1; done
for prec in fp32 fp64; do timeout 300 python tools/prof_run.py $prec 200 200 2>&1 | tail -1; done
