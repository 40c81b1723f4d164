timeout 300 python tools/single_chain.py > gpurun_out/sc1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t43.log 2>&1
