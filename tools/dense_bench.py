"""Config-4 shape probe: dense Gaussian D=1000, C chains in lockstep.
Usage: python tools/dense_bench.py [tf32|fp64] [C] [W] [S] [D]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1912_11554_b200 as ts

prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
W = int(sys.argv[3]) if len(sys.argv) > 3 else 100
S = int(sys.argv[4]) if len(sys.argv) > 4 else 100
D = int(sys.argv[5]) if len(sys.argv) > 5 else 1000
rng = np.random.default_rng(4)
q, _ = np.linalg.qr(rng.standard_normal((D, D)))
lam = np.logspace(-2, 2, D)
Sigma = (q * lam) @ q.T
P = (q / lam) @ q.T
for dense_mass in ((True,) if os.environ.get("DENSE_ONLY_MASS") else ((False,) if os.environ.get("DENSE_NO_MASS") else (False, True))):
    m = ts.dense_gaussian_model(P, inv_mass=Sigma if dense_mass else None, precision=prec)
    cfg = ts.RunConfig(model={}, num_chains=C, num_warmup=W, num_samples=S, seed=4)
    for it in range(2):
        r = ts.run_device(m, cfg, ts.chain_keys(4, C), 0)
        st = r.stats.cpu().numpy()
        lf = st[:, :, 1].sum()
        ev = r.evals.cpu().numpy()
        steps = ev.max()
        print(f"{prec} dense_mass={dense_mass} D={D} C={C} W={W} S={S}: {r.event_ms:.1f} ms, {lf:.0f} chain-leapfrogs "
              f"({lf / (r.event_ms / 1e3) / 1e6:.2f} M/s), lockstep steps {steps}, {r.event_ms * 1e3 / steps:.1f} us/step, "
              f"GEMM {2.0 * D * D * C * steps / (r.event_ms / 1e3) / 1e12:.1f} TFLOP/s, mean depth {st[:, W:, 0].mean():.2f}",
              flush=True)
