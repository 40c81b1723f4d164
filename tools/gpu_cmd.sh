python tools/check_pathology.py 1 > gpurun_out/patho.log 2>&1
