"""Config 1 probe: 10-D Gaussian, one chain, thread vs block team."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1912_11554_b200 as ts
m = ts.gaussian_model(np.ones(10))
cfg = ts.RunConfig(model={}, num_chains=1, num_warmup=1000, num_samples=1000, seed=7)
for mode in ("thread", "block", "thread", "block"):
    r = ts.run_device(m, cfg, ts.chain_keys(7, 1), 0, exec_mode=mode)
    lf = float(r.stats.cpu().numpy()[:, :, 1].sum())
    print(f"{mode}: {r.event_ms:.1f} ms, {lf:.0f} leapfrogs, {lf / (r.event_ms / 1e3):.0f} leapfrog/s", flush=True)
