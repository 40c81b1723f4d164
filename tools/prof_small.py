"""TS_PROF cycle counters of a one-chain small-model run in a warp team
(usage: TS_PROF=1 python tools/prof_small.py [gauss10|eight_schools])."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1912_11554_b200 as ts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gauss10"
model = ts.gaussian_model(np.ones(10)) if name == "gauss10" else ts.eight_schools_model()
cfg = ts.RunConfig(model={}, num_chains=1, num_warmup=1000, num_samples=1000, seed=7)
for mode in ("warp",):
    r = ts.run_device(model, cfg, ts.chain_keys(7, 1), 0, exec_mode=mode)
    torch.cuda.synchronize()
    lf = float(r.stats.cpu().numpy()[:, :, 1].sum())
    print(mode, "ms", r.event_ms, "leapfrogs", lf, "us/lf", r.event_ms * 1000 / lf, flush=True)
