"""Debug: device runs (thread team) vs the reference golden runs, every record."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1912_11554_b200 as t
recs = json.load(open(os.path.join(ROOT, "tests/golden/runs.json")))
for k, rec in enumerate(recs):
    desc = dict(rec["desc"])
    model = t.eight_schools_model() if desc["model"] == "eight_schools" else t.model_from_descriptor(desc)
    sampler = None
    if rec["sampler"] is not None:
        s = rec["sampler"]
        sampler = t.SamplerConfig(step_size=s["step"], mass=t.MassMatrix.identity(model.dim), criterion=s["criterion"], max_tree_depth=s["max_tree_depth"])
    cfg = t.RunConfig(model=desc, num_chains=rec["num_chains"], num_warmup=rec["num_warmup"], num_samples=rec["num_samples"], seed=rec["seed"], sampler=sampler)
    for mode in ("thread", "warp", None):
        res = t.run(cfg, model, exec_mode=mode)
        for ci, (r, ref) in enumerate(zip(res, rec["chains"])):
            rs = np.asarray([[float(v) for v in s] for s in ref["stats"]])
            bad = np.nonzero((r.stats_array[:, :3] != rs[:, :3]).any(1))[0]
            sm = np.asarray([[float(v) for v in s] for s in ref["samples"]])
            print(k, desc["model"], rec["num_warmup"], mode, "chain", ci, "stat mismatches", bad[:4], "max |dq|", float(np.abs(r.samples - sm).max()),
                  "step", r.adaptation["final_step_size"], float(ref["adaptation"]["final_step_size"]))
