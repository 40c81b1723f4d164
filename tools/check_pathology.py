"""Do long (depth-10) sampling transitions of the covtype run reproduce on the
CPU oracle?  Re-runs transition i of a device run from the device's own state
on both the device and the oracle (fp64) and compares the decisions."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1912_11554_b200 as ts
import turnstile_oracle as o
from tests_data import logistic_data

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
x, y = logistic_data(581012, 54, 20191222)
m = ts.logistic_regression_model(ts.LogisticRegressionData(x.astype(np.float32), y), precision="fp64")
W, S = 1000, 1000
cfg = ts.RunConfig(model={}, num_chains=1, num_warmup=W, num_samples=S, seed=seed)
key = ts.chain_keys(seed, 1)[0]
r = ts.run_device(m, cfg, [key], 0)
st = r.stats.cpu().numpy()[0]; ad = r.adapt.cpu().numpy()[0]; samples = r.samples.cpu().numpy()[0]
step, inv = float(ad[1]), ad[2 + W:].copy()
deep = [i for i in range(1, S) if st[W + i, 0] >= 9][:2]
shallow = [i for i in range(1, S) if st[W + i, 0] <= 3][:1]
om = o.Model("logistic_regression", 55, x=x, y=y, fused_omp=True)
print("depth hist", np.bincount(st[W:, 0].astype(int), minlength=11).tolist(), "step", step, flush=True)
qs = samples[::50]
print("U along the sampling phase:", [round(m.potential(q), 1) for q in qs[:20]], flush=True)
for i in deep + shallow:
    q0 = samples[i - 1]
    U0 = m.potential(q0); g0 = m.gradient(q0)
    z = ts.PhasePoint(q0, np.zeros(55), U0, g0)
    sc = ts.SamplerConfig(step_size=step, mass=ts.MassMatrix(inv))
    dkey = key.fold(10 + W + i)
    z1, s1 = ts.nuts_transition_from(z, sc, m, dkey)
    t0 = time.time()
    oz, os_, dec = o.transition(o.Point(q0.tolist(), [0.0] * 55, U0, g0.tolist()), step, inv.tolist(), om,
                                (dkey.hi, dkey.lo))
    print(f"draw {i}: device depth={s1.depth_reached} lf={s1.leapfrog_calls} | run depth={int(st[W+i,0])} "
          f"lf={int(st[W+i,1])} | oracle depth={os_.depth} lf={os_.leapfrogs} ({time.time()-t0:.0f}s) "
          f"|dq|={np.abs(z1.position - np.asarray(oz.q)).max():.2e}", flush=True)
