mkdir -p gpurun_out
for ns in 2 3; do for k in 50 70 85; do echo "fp32 NSTAGE=$ns KEEP=$k: $(TS_NSTAGE=$ns TS_L2_KEEP=$k timeout 120 python tools/prof_eval.py fp32 200 | tail -1 | cut -c1-90) | $(TS_NSTAGE=$ns TS_L2_KEEP=$k timeout 200 python tools/prof_run.py fp32 200 200 2>&1 | tail -1 | cut -c40-100)"; done; done
for k in 0 30 60; do echo "fp64 KEEP=$k: $(TS_L2_KEEP=$k timeout 120 python tools/prof_eval.py fp64 100 | tail -1 | cut -c1-90)"; done
for k in 0 20 35; do echo "fp64x KEEP=$k: $(TS_L2_KEEP=$k timeout 120 python tools/prof_eval.py fp64x 100 | tail -1 | cut -c1-90)"; done
