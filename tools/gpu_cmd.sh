timeout 600 python -m pytest tests -m gpu -q -x -k "row_shard or wide" > gpurun_out/t50.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t51.log 2>&1
