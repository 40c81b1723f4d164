"""Many-chain covtype logistic on the tensor cores (precision tf32): chain-leapfrog/s.
Usage: python tools/lm_bench.py C [W] [S]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data_f32
C = int(sys.argv[1]) if len(sys.argv) > 1 else 256
W = int(sys.argv[2]) if len(sys.argv) > 2 else 100
S = int(sys.argv[3]) if len(sys.argv) > 3 else 100
x, y = logistic_data_f32(581012, 54, 20191222)
m = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision="tf32")
cfg = ts.RunConfig(model={}, num_chains=C, num_warmup=W, num_samples=S, seed=1)
keys = ts.chain_keys(1, C)
for it in range(2):
    r = ts.run_device(m, cfg, keys, 0)
    st = r.stats.cpu().numpy()
    lf = float(st[:, :, 1].sum())
    steps = float(r.evals.cpu().numpy().max())
    e, rh = ts.chain_diagnostics_device(r.samples)
    print(f"C={C} W={W} S={S}: {r.event_ms:.1f} ms, {lf:.0f} chain-leapfrogs -> {lf / r.event_ms * 1e3 / 1e6:.3f} M/s, "
          f"max evals/chain {steps:.0f}, {r.event_ms * 1e3 / max(steps, 1):.1f} us per chain-eval, min ESS {np.nanmin(e):.0f}, "
          f"ESS/s {np.nanmin(e) / r.event_ms * 1e3:.1f}, max R-hat {np.nanmax(rh):.3f}", flush=True)
