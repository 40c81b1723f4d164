nvidia-smi -L > gpurun_out/smi.txt
timeout 1500 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/t.log 2>&1; echo tests=$?
tail -15 gpurun_out/t.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -c 3000 gpurun_out/bench.json
