# round-2 evidence batch: bench line, launch list, ncu captures (summarised on the box), flip log
mkdir -p gpurun_out
S0=$(date +%s)
timeout 1500 python -m pytest tests/ -q -rP -m gpu -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo tests=$?; tail -2 gpurun_out/tall.log; grep -o "dense tf32 decision replay: .\{0,120\}" gpurun_out/tall.log
S0=$(date +%s)
timeout 2400 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench=$? wall=$(( $(date +%s) - S0 ))s
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r2.json").read().strip().splitlines()[-1])
print("value", d["value"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"], "cpu", d.get("cpu_baseline", {}).get("value"))
for k, v in d.items():
    if isinstance(v, dict) and "wall_s_rank0" in v:
        print(k, "wall", round(v["wall_s_rank0"], 1), "value", v.get("value"), "cpu", (v.get("cpu_baseline") or {}).get("value"), v.get("error", ""))
PY
TS_FLIP_LOG=gpurun_out/r2_fp32_flips.json timeout 900 python -m pytest tests/test_gpu_covtype_fp32.py -q -s -p no:cacheprovider -k "replay" > gpurun_out/flips.log 2>&1; echo flips=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 1 --warmup 0 --subs '' --no-cpu --no-e2e --num-warmup 20 --num-samples 10 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
for prec in fp32 fp64; do
  timeout 300 python tools/prof_run.py $prec 60 40 > gpurun_out/prof_run_$prec.log 2>&1; tail -1 gpurun_out/prof_run_$prec.log
  P=$(grep -o "[0-9]* passes" gpurun_out/prof_run_$prec.log | tail -1 | cut -d' ' -f1)
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_block_op --launch-skip 1 -c 1 -o /tmp/r2_run_$prec -f python tools/prof_run.py $prec 60 40 > gpurun_out/ncu_r2run_$prec.log 2>&1; echo ncu_$prec=$?
  python tools/ncu_summary.py /tmp/r2_run_$prec.ncu-rep gpurun_out/r2_ncu_run_$prec.json $P > /dev/null
  ncu -i /tmp/r2_run_$prec.ncu-rep --page source --csv --print-source sass > /tmp/src_$prec.csv 2>/dev/null; python tools/sass_regions.py /tmp/src_$prec.csv > gpurun_out/r2_run_${prec}_regions.txt 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:k_dense_op --launch-skip 1 -c 1 -o /tmp/r2_dense -f env DENSE_ONLY_MASS=1 python tools/dense_bench.py tf32 1024 20 10 > gpurun_out/ncu_dense.log 2>&1; echo ncudense=$?
python tools/ncu_summary.py /tmp/r2_dense.ncu-rep gpurun_out/r2_ncu_dense_raw.json > /dev/null
ls -la gpurun_out
