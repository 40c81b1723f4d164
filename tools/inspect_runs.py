"""Per-run adaptation/tree-depth summary for a few seeds (diagnostic)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1912_11554_b200 as ts
from tests_data import logistic_data
x, y = logistic_data(581012, 54, 20191222)
for prec in sys.argv[1].split(","):
    m = ts.logistic_regression_model(ts.LogisticRegressionData(x.astype(np.float32), y), precision=prec)
    for seed in [int(s) for s in sys.argv[2].split(",")]:
        cfg = ts.RunConfig(model={}, num_chains=1, num_warmup=1000, num_samples=1000, seed=seed)
        r = ts.run_device(m, cfg, ts.chain_keys(seed, 1), 0)
        st = r.stats.cpu().numpy()[0]; ad = r.adapt.cpu().numpy()[0]
        W = 1000
        depth = st[:, 0].astype(int); lf = st[:, 1]
        print(f"{prec} seed={seed}: {r.event_ms:.0f} ms, lf warm={lf[:W].sum():.0f} samp={lf[W:].sum():.0f}, "
              f"eps0={ad[0]:.3g} final_eps={ad[1]:.3g} inv_mass[min,max]=({ad[2+W:].min():.3g},{ad[2+W:].max():.3g}) "
              f"depth hist samp={np.bincount(depth[W:], minlength=11).tolist()} div={int(st[:,2].sum())} "
              f"accept samp={st[W:,3].mean():.3f}", flush=True)
