# summarise the r2 evidence batch into profiles/
set -x
P32=$(grep -o "[0-9]* passes" gpurun_out/prof_run_fp32.log | tail -1 | cut -d' ' -f1)
P64=$(grep -o "[0-9]* passes" gpurun_out/prof_run_fp64.log | tail -1 | cut -d' ' -f1)
python tools/ncu_summary.py gpurun_out/r2_run_fp32.ncu-rep profiles/r2_ncu_run_fp32.json $P32 > /dev/null
python tools/ncu_summary.py gpurun_out/r2_run_fp64.ncu-rep profiles/r2_ncu_run_fp64.json $P64 > /dev/null
python tools/ncu_summary.py gpurun_out/r2_dense.ncu-rep /tmp/r2_dense.json > /dev/null
python tools/ncu_summary.py gpurun_out/r2_many.ncu-rep /tmp/r2_many.json > /dev/null
cp gpurun_out/bench_r2.json profiles/r2_bench_line.json
cp gpurun_out/r2_launches_bench.csv profiles/r2_launches_bench.csv
cp gpurun_out/r2_fp32_flips.json profiles/r2_fp32_flips.json 2>/dev/null
