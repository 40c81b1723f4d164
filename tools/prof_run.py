"""Profiling driver: a short logistic NUTS run (one persistent launch).
Usage: python tools/prof_run.py [fp64|fp32] [num_warmup] [num_samples] [N] [p] [seed]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data_f32

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 60
S = int(sys.argv[3]) if len(sys.argv) > 3 else 40
N = int(sys.argv[4]) if len(sys.argv) > 4 else 581012
P = int(sys.argv[5]) if len(sys.argv) > 5 else 54
seed = int(sys.argv[6]) if len(sys.argv) > 6 else 20191222
x, y = logistic_data_f32(N, P, seed)
m = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision=prec)
RUN_SEED = int(os.environ.get("RUN_SEED", "1"))
cfg = ts.RunConfig(model={}, num_chains=1, num_warmup=W, num_samples=S, seed=RUN_SEED)
algo = 4 * N * P + N
for it in range(2):
    r = ts.run_device(m, cfg, ts.chain_keys(RUN_SEED, 1), 0)
    lf = float(r.stats.cpu().numpy()[0][:, 1].sum()); ev = float(r.evals.cpu().numpy()[0])
    print(f"{prec} {N}x{P} run W={W} S={S}: {r.event_ms:.1f} ms, {lf:.0f} leapfrogs, {ev:.0f} passes, "
          f"{r.event_ms*1000/lf:.2f} us/leapfrog, {algo*ev/(r.event_ms/1e3)/1e9:.0f} GB/s", flush=True)
