"""Debug: first mismatch between a device run (thread team) and the reference golden run."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1912_11554_b200 as t
import turnstile_oracle as o
recs = json.load(open(os.path.join(ROOT, "tests/golden/runs.json")))
num = lambda v: float(v) if not isinstance(v, str) else float(v)
for rec in recs:
    if rec["num_warmup"] == 0:
        continue
    desc = dict(rec["desc"])
    model = t.eight_schools_model() if desc["model"] == "eight_schools" else t.model_from_descriptor(desc)
    cfg = t.RunConfig(model=desc, num_chains=rec["num_chains"], num_warmup=rec["num_warmup"], num_samples=rec["num_samples"], seed=rec["seed"])
    res = t.run(cfg, model, exec_mode="thread")
    md = {"name": desc["model"], **desc.get("params", {})}
    om = o.model_from_desc(md)
    for ci, (r, ref) in enumerate(zip(res, rec["chains"])):
        key = o.chain_keys(rec["seed"], rec["num_chains"])[ci]
        out = o.run_chain(om, key, rec["num_warmup"], rec["num_samples"])
        ow = np.asarray([[s.depth, s.leapfrogs, int(s.diverged), s.accept, s.energy] for s in out["stats"]])
        dv = np.vstack([r.warmup_stats_array, r.stats_array])
        tr_d = np.asarray(r.adaptation["step_size_trace"]); tr_o = np.asarray(out["adaptation"]["step_size_trace"])
        print(desc["model"], "chain", ci, "eps0", r.adaptation["initial_step_size"], out["adaptation"]["initial_step_size"])
        bad = np.nonzero((dv[:, :3] != ow[:, :3]).any(1) | (np.abs(dv[:, 3:] - ow[:, 3:]) > 1e-12 * np.abs(ow[:, 3:]) + 1e-300).any(1))[0]
        tbad = np.nonzero(tr_d != tr_o)[0]
        print("  first stat mismatch draw", bad[:3], " first step-trace mismatch", tbad[:3])
        if tbad.size:
            i = tbad[0]; print("  step", i, repr(tr_d[i]), repr(tr_o[i]), "prev accept dev/or", dv[i-1, 3] if i else None, ow[i-1, 3] if i else None)
        if bad.size:
            i = bad[0]; print("  draw", i, dv[i].tolist(), ow[i].tolist())
