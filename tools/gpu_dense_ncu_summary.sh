#!/bin/bash
# ncu --set full of one config-4 run (second launch of tools/dense_bench.py tf32 1024 20 10),
# summarised on the box into gpurun_out/r2_ncu_dense.json (the report stays in /tmp)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:k_dense_op --launch-skip 1 -c 1 -o /tmp/dn -f \
  env DENSE_ONLY_MASS=1 python tools/dense_bench.py tf32 1024 20 10 > gpurun_out/ncu_dn.log 2>&1; echo ncu=$?
python tools/ncu_summary.py /tmp/dn.ncu-rep /tmp/dn_raw.json > /dev/null 2>&1
python - <<'PY'
import json, re
raw = json.load(open("/tmp/dn_raw.json"))[0]
log = open("gpurun_out/ncu_dn.log").read()
lf = [float(x) for x in re.findall(r"([0-9]+) chain-leapfrogs", log)]
chain_lf = lf[-1] if lf else None
dram = raw.get("dram__bytes_read.sum", 0) * 1e9 / 1e9
def b(k):
    v = raw.get(k); u = raw.get(k + ".unit", "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return v * scale if v is not None else None
dram_bytes = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
out = {"kernel": raw["kernel"],
       "command": "ncu --set full --clock-control none -k regex:k_dense_op --launch-skip 1 -c 1 env DENSE_ONLY_MASS=1 python tools/dense_bench.py tf32 1024 20 10",
       "tensor_pipe_pct": raw.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
       "issue_active_pct": raw.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
       "warps_active_pct": raw.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
       "l2_hit_pct": raw.get("lts__t_sector_hit_rate.pct"),
       "stall_barrier_per_issue": raw.get("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
       "stall_long_scoreboard_per_issue": raw.get("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
       "dram_bytes": dram_bytes, "chain_leapfrogs": chain_lf,
       "dram_bytes_per_chain_leapfrog": dram_bytes / chain_lf if chain_lf else None,
       "registers": raw.get("launch__registers_per_thread"), "grid": raw.get("launch__grid_size"),
       "block": raw.get("launch__block_size"),
       "note": "cooperative kernel whose warps spin on cross-CTA flags: under ncu replay durations are not meaningful; pipe percentages are per active cycle"}
json.dump(out, open("gpurun_out/r2_ncu_dense.json", "w"), indent=1)
print(json.dumps(out)[:600])
PY
