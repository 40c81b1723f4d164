"""Profiling driver: a short covtype-shaped NUTS run (one persistent launch).
Usage: python tools/prof_run.py [fp64|fp32] [num_warmup] [num_samples]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 60
S = int(sys.argv[3]) if len(sys.argv) > 3 else 40
x, y = logistic_data(581012, 54, 20191222)
m = ts.logistic_regression_model(ts.LogisticRegressionData(x.astype(np.float32), y), precision=prec)
cfg = ts.RunConfig(model={}, num_chains=1, num_warmup=W, num_samples=S, seed=1)
for it in range(2):
    r = ts.run_device(m, cfg, ts.chain_keys(1, 1), 0)
    lf = float(r.stats.cpu().numpy()[0][:, 1].sum()); ev = float(r.evals.cpu().numpy()[0])
    print(f"{prec} run W={W} S={S}: {r.event_ms:.1f} ms, {lf:.0f} leapfrogs, {ev:.0f} passes, "
          f"{r.event_ms*1000/lf:.2f} us/leapfrog", flush=True)
