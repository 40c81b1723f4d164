timeout 900 python -m pytest tests -m gpu -q -x -k "dense or tcgen05 or row_shard or wide" > gpurun_out/t40.log 2>&1
