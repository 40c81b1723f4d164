"""Scratch diagnostics for GPU parity (prints max diffs); not a test."""
import sys, json, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle'); sys.path.insert(0,'tests')
import paper_1912_11554_b200 as t, turnstile_oracle as o
from conftest import golden, num, nums
m = t.eight_schools_model(); om = o.model_from_desc({"name":"eight_schools"})
pts = np.random.default_rng(3).standard_normal((6, 10))*1.3
out = t.models.potential_and_gradient(m.device_spec, pts)
for k in range(6):
    q = pts[k].tolist(); g = np.asarray(om.gradient(q))
    d = out[k,1:] - g
    print("8s", k, out[k,0]-om.potential(q), np.nonzero(d)[0], d[np.nonzero(d)[0]])
for rec in golden("runs")[:2]:
    desc = rec["desc"]; model = t.model_from_descriptor(desc)
    cfg = t.RunConfig(model=desc, num_chains=rec["num_chains"], num_warmup=rec["num_warmup"], num_samples=rec["num_samples"], seed=rec["seed"])
    res = t.run(cfg, model)
    for r, ref in zip(res, rec["chains"]):
        rs = np.asarray([nums(s) for s in ref["samples"]])
        d = np.abs(r.samples - rs)
        print("run", desc["model"], "maxdiff", d.max(), "first draw with diff", np.nonzero(d.max(axis=1) > 0)[0][:5])
        print(" step", r.adaptation["final_step_size"], num(ref["adaptation"]["final_step_size"]), r.adaptation["initial_step_size"], num(ref["adaptation"]["initial_step_size"]))
        tr = np.asarray(r.adaptation["step_size_trace"]); rtr = np.asarray(nums(ref["adaptation"]["step_size_trace"]))
        print(" trace first diff", np.nonzero(tr != rtr)[0][:5], "max rel", np.max(np.abs(tr-rtr)/rtr))
        print(" inv", np.max(np.abs(np.asarray(r.adaptation["inv_mass_diag"]) - nums(ref["adaptation"]["inv_mass_diag"]))))
        print(" stats accept maxdiff", np.max(np.abs(r.stats_array[:,3] - [num(s[3]) for s in ref["stats"]])))
        print(" samples[0]", r.samples[0][:3], rs[0][:3])
