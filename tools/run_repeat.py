"""Repeated covtype runs in one process: per-run time, passes, nvidia-smi clocks/power after each run.
Usage: python tools/run_repeat.py [n_runs] [sleep_s] [seed]"""
import os, sys, time, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data_f32
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
gap = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1001
x, y = logistic_data_f32(581012, 54, 20191222)
m = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision="fp32")
cfg = ts.RunConfig(model={}, num_chains=1, num_warmup=1000, num_samples=1000, seed=seed)
def smi():
    q = "clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
for i in range(n):
    r = ts.run_device(m, cfg, ts.chain_keys(seed, 1), 0)
    ev = float(r.evals.cpu().numpy()[0])
    print(f"run {i}: {r.event_ms:.1f} ms, {ev:.0f} passes, {r.event_ms * 1e3 / ev:.2f} us/pass | {smi()}", flush=True)
    if gap: time.sleep(gap)
