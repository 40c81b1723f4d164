"""Generate golden fixtures by running the REFERENCE (turnstile) in this container.

Usage (from the repo root, where /root/reference exists):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src and run on
its default (numba) kernel path.  Outputs, committed under tests/golden/:
  rng.json          RngKey.from_seed/split/fold words, uniform and normal streams
  trees.json        build_tree_iterative cases (crosscheck.build_case
                    distribution + the test_trees.py schedule cases): inputs,
                    Tree fields, TreeTrace, proposal leaf index
  transitions.json  nuts_transition_from chains of draws with per-tree
                    decisions (direction, leapfrogs, stop, proposal leaf)
  runs.json         full run() results (samples, stats, adaptation) for small
                    models, incl. eight-schools through the TargetModel plugin API
  logistic.json     logistic potential/gradient at fixed points (fp32-exact data)
  hmc.json          hmc_transition chains (fixed-length HMC baseline, sampler.py:163-203)
Nothing here is read by the GPU box at run time except these JSON files.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import turnstile  # noqa: E402
from turnstile import chains as tchains  # noqa: E402
from turnstile import sampler as tsampler  # noqa: E402
from turnstile import tree as ttree  # noqa: E402
from turnstile.crosscheck import build_case  # noqa: E402
from turnstile.integrator import MassMatrix, PhasePoint, hamiltonian  # noqa: E402
from turnstile.models import (  # noqa: E402
    LogisticRegressionData,
    TargetModel,
    funnel_model,
    gaussian_model,
    logistic_regression_model,
    std_normal_model,
)
from turnstile.rng import RngKey  # noqa: E402
from turnstile.sampler import SamplerConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f(x):
    """JSON-safe float (inf/nan as strings), exact via repr round trip."""
    x = float(x)
    if math.isnan(x):
        return "nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return x


def fl(a):
    return [f(v) for v in np.asarray(a, dtype=np.float64).ravel().tolist()]


def model_desc(model):
    """Serializable description of a reference model built by build_case."""
    if model.name == "std_normal":
        return {"name": "std_normal", "dim": model.dim}
    if model.name == "gaussian":
        return {"name": "gaussian", "cov_diag": fl(model.params["cov_diag"])}
    if model.name == "funnel":
        return {"name": "funnel", "dim": model.dim}
    if model.name == "logistic_regression":
        # recover the closure data
        cells = {c.cell_contents.__class__.__name__: c.cell_contents for c in model.potential.__closure__ or []}
        x = y = None
        for c in model.potential.__closure__:
            v = c.cell_contents
            if isinstance(v, np.ndarray) and v.ndim == 2:
                x = v
            elif isinstance(v, np.ndarray) and v.ndim == 1:
                y = v
        return {"name": "logistic_regression", "x": [fl(r) for r in x], "y": fl(y)}
    raise ValueError(model.name)


class LeafRecorder:
    """Rebinds turnstile.tree.leapfrog to collect the leaves in generation order."""

    def __init__(self):
        self.leaves = []
        self._orig = ttree.leapfrog

    def __enter__(self):
        def rec(*a, **k):
            z = self._orig(*a, **k)
            self.leaves.append(z)
            return z

        ttree.leapfrog = rec
        return self

    def __exit__(self, *exc):
        ttree.leapfrog = self._orig


def leaf_index(leaves, z):
    for i, l in enumerate(leaves):
        if l is z:
            return i
    return -1


def tree_record(z, depth, eps, config, model, key, h_ref=None):
    trace = ttree.TreeTrace()
    with LeafRecorder() as rec:
        t = ttree.build_tree_iterative(z, depth, eps, config, model, key, h_ref=h_ref, trace=trace)
    return {
        "model": model_desc(model),
        "z": {"q": fl(z.position), "r": fl(z.momentum), "U": f(z.potential), "g": fl(z.grad)},
        "depth": depth,
        "eps": f(eps),
        "h_ref": f(hamiltonian(z, config.mass) if h_ref is None else h_ref),
        "inv_diag": fl(config.mass.inv_diag),
        "criterion": config.criterion,
        "max_tree_depth": config.max_tree_depth,
        "threshold": f(config.divergence_threshold),
        "key": [str(key.hi), str(key.lo)],
        "out": {
            "left_q": fl(t.left.position), "left_r": fl(t.left.momentum), "left_U": f(t.left.potential),
            "right_q": fl(t.right.position), "right_r": fl(t.right.momentum), "right_U": f(t.right.potential),
            "right_g": fl(t.right.grad),
            "prop_q": fl(t.proposal.position), "prop_U": f(t.proposal.potential), "prop_g": fl(t.proposal.grad),
            "prop_H": f(hamiltonian(t.proposal, config.mass)),
            "log_weight": f(t.log_weight), "turning": t.turning, "diverging": t.diverging,
            "leapfrog_count": t.leapfrog_count, "momentum_sum": fl(t.momentum_sum),
            "sum_metropolis": f(t.sum_metropolis),
            "proposal_leaf": leaf_index(rec.leaves, t.proposal),
        },
        "trace": {
            "writes": trace.writes, "checks": [list(c) for c in trace.checks],
            "leaf_log_weights": fl(trace.leaf_log_weights), "max_occupied": trace.max_occupied,
        },
    }


def gen_trees():
    cases = []
    root = RngKey.from_seed(20240809)
    for depth in range(0, 9):
        for trial in range(12):
            case_key = root.fold(depth * 1_000_000 + trial)
            z, eps, config, model = build_case(case_key, depth, trial)
            cases.append(tree_record(z, depth, eps, config, model, case_key.fold(1)))
    # schedule cases from the reference tests (test_trees.py:150-222, test_acceptance.py:81-97)
    m2 = std_normal_model(2)
    cfg = SamplerConfig(step_size=1e-3, mass=MassMatrix.identity(2), max_tree_depth=4)
    z = PhasePoint.from_position(m2, [0.4, -0.1], [0.8, 0.6])
    cases.append(tree_record(z, 4, 1e-3, cfg, m2, RngKey.from_seed(11)))
    gen = RngKey.from_seed(3).fold(0).generator()
    zq, zr = gen.standard_normal(2), gen.standard_normal(2)
    z = PhasePoint.from_position(m2, zq, zr)
    cfg = SamplerConfig(step_size=0.6, mass=MassMatrix.identity(2), max_tree_depth=12)
    cases.append(tree_record(z, 10, 0.6, cfg, m2, RngKey.from_seed(5)))
    # divergent (test_trees.py:252-263) and a backward deep tree
    m1 = std_normal_model(1)
    cfgd = SamplerConfig(step_size=5.0, mass=MassMatrix.identity(1), max_tree_depth=8, divergence_threshold=50.0)
    for seed in range(3):
        g = RngKey.from_seed(seed).fold(0).generator()
        z = PhasePoint.from_position(m1, g.standard_normal(1) * 3, g.standard_normal(1) * 8)
        cases.append(tree_record(z, 8, 5.0, cfgd, m1, RngKey.from_seed(seed).fold(1)))
    m3 = gaussian_model([0.5, 2.0, 1.0])
    for crit in ("classic", "generalized"):
        cfg3 = SamplerConfig(step_size=0.4, mass=MassMatrix.identity(3), max_tree_depth=12, criterion=crit)
        g = RngKey.from_seed(77).fold(0).generator()
        z = PhasePoint.from_position(m3, g.standard_normal(3), g.standard_normal(3))
        for sign in (1.0, -1.0):
            cases.append(tree_record(z, 8, sign * 0.4, cfg3, m3, RngKey.from_seed(31)))
    # full-depth tiny-step trees: R-slot high-water mark (test_trees.py:191-200)
    for depth in (6, 10):
        cfgs = SamplerConfig(step_size=1e-4, mass=MassMatrix.identity(2), max_tree_depth=12)
        g = RngKey.from_seed(21).fold(0).generator()
        z = PhasePoint.from_position(m2, g.standard_normal(2) * 0.3, g.standard_normal(2))
        cases.append(tree_record(z, depth, 1e-4, cfgs, m2, RngKey.from_seed(2)))
    return cases


def gen_transitions():
    out = []
    specs = [
        (std_normal_model(10), "generalized", 0.9, 10, 101),
        (gaussian_model(np.logspace(-1, 1, 5)), "classic", 0.3, 10, 102),
        (funnel_model(6), "generalized", 0.4, 8, 103),
        (gaussian_model([0.5, 2.0, 1.0]), "generalized", 1.3, 6, 104),
    ]
    for model, crit, step, mtd, seed in specs:
        mass = MassMatrix(np.linspace(0.7, 1.4, model.dim))
        cfg = SamplerConfig(step_size=step, mass=mass, max_tree_depth=mtd, criterion=crit)
        key = RngKey.from_seed(seed)
        z = PhasePoint.from_position(model, key.fold(0).generator().uniform(-1, 1, model.dim), np.zeros(model.dim))
        draws = []
        for i in range(12):
            dkey = key.fold(10 + i)
            trees, outer = [], []
            orig_build, orig_check = tsampler.build_tree_iterative, tsampler.check_uturn

            def build(frontier, j, eps, config, model_, rng, h_ref=None, trace=None):
                with LeafRecorder() as rec:
                    t = orig_build(frontier, j, eps, config, model_, rng, h_ref=h_ref)
                trees.append([j, 1 if eps > 0 else 0, t.leapfrog_count, int(t.turning), int(t.diverging),
                              leaf_index(rec.leaves, t.proposal)])
                return t

            def check(*a, **k):
                r = orig_check(*a, **k)
                outer.append(int(r))
                return r

            tsampler.build_tree_iterative = build
            tsampler.check_uturn = check
            try:
                z_in = z
                z, stats = turnstile.nuts_transition_from(z, cfg, model, dkey)
            finally:
                tsampler.build_tree_iterative, tsampler.check_uturn = orig_build, orig_check
            draws.append({
                "key": [str(dkey.hi), str(dkey.lo)],
                "z_in": {"q": fl(z_in.position), "U": f(z_in.potential), "g": fl(z_in.grad)},
                "z_out": {"q": fl(z.position), "U": f(z.potential), "g": fl(z.grad)},
                "stats": [stats.depth_reached, stats.leapfrog_calls, int(stats.diverged), f(stats.accept_stat),
                          f(stats.energy)],
                "trees": trees,
                "outer": outer,
            })
        out.append({"model": model_desc(model), "criterion": crit, "step": step, "max_tree_depth": mtd,
                    "inv_diag": fl(mass.inv_diag), "draws": draws})
    return out


def eight_schools_twin():
    """Eight schools NC through the reference's plugin API (oracle twin,
    same op order as oracle/turnstile_oracle.py and csrc/ts_models.cuh)."""
    y = [28.0, 8.0, -3.0, 7.0, -1.0, 1.0, 18.0, 12.0]
    s = [15.0, 10.0, 16.0, 11.0, 9.0, 11.0, 10.0, 18.0]
    sys.path.insert(0, os.path.join(os.path.dirname(OUT), "..", "oracle"))
    from turnstile_oracle import eight_schools_potential, eight_schools_gradient

    return TargetModel("eight_schools", 10, lambda q: eight_schools_potential(q, y, s),
                       lambda q: eight_schools_gradient(q, y, s), {"y": y, "sigma": s})


def gen_runs():
    out = []
    specs = [
        ({"model": "std_normal", "params": {"dim": 10}}, None, 2, 150, 150, 7, None),
        ({"model": "gaussian", "params": {"cov_diag": np.logspace(-2, 2, 10).tolist()}}, None, 1, 200, 100, 11, None),
        ({"model": "funnel", "params": {"dim": 4}}, None, 1, 40, 30, 5, None),
        ({"model": "eight_schools", "params": {}}, "eight", 3, 100, 50, 3, None),
        ({"model": "std_normal", "params": {"dim": 3}}, None, 2, 0, 40, 9, None),
        ({"model": "std_normal", "params": {"dim": 3}}, None, 1, 0, 40, 9, ("classic", 0.7, 5)),
    ]
    for desc, special, C, W, S, seed, samp in specs:
        model = eight_schools_twin() if special == "eight" else turnstile.model_from_descriptor(desc)
        sampler = None
        if samp is not None:
            sampler = SamplerConfig(step_size=samp[1], mass=MassMatrix.identity(model.dim), criterion=samp[0],
                                    max_tree_depth=samp[2])
        cfg = tchains.RunConfig(model=desc, num_chains=C, num_warmup=W, num_samples=S, seed=seed, sampler=sampler)
        res = tchains.run(cfg, model)
        out.append({
            "desc": desc, "num_chains": C, "num_warmup": W, "num_samples": S, "seed": seed,
            "sampler": None if samp is None else {"criterion": samp[0], "step": samp[1], "max_tree_depth": samp[2]},
            "chains": [{
                "samples": [fl(row) for row in r.samples],
                "stats": [[s.depth_reached, s.leapfrog_calls, int(s.diverged), f(s.accept_stat), f(s.energy)]
                          for s in r.stats],
                "total_leapfrogs": r.total_leapfrogs,
                "adaptation": {k: (fl(v) if isinstance(v, (list, np.ndarray)) else f(v)) for k, v in r.adaptation.items()},
            } for r in res],
        })
    return out


sys.path.insert(0, os.path.join(OUT, ".."))
from tests_data import logistic_data  # noqa: E402


def gen_logistic():
    out = []
    for n, p, seed in ((37, 3, 1), (1000, 54, 2), (4099, 54, 3), (777, 20, 4), (50, 64, 5)):
        x, yv = logistic_data(n, p, seed)
        model = logistic_regression_model(LogisticRegressionData(x, yv))
        g = np.random.default_rng(seed + 100)
        pts = [np.zeros(p + 1), g.standard_normal(p + 1) * 0.1, g.standard_normal(p + 1) * 3.0]
        out.append({
            "n": n, "p": p, "seed": seed,
            "points": [{"q": fl(q), "U": f(model.potential(q)), "g": fl(model.gradient(q))} for q in pts],
        })
    return out


def gen_rng():
    out = {"seeds": []}
    for seed in (0, 1, 7, 20191222, 2**70 + 5):
        k = RngKey.from_seed(seed)
        a, b = k.split()
        rec = {
            "seed": str(seed), "key": [str(k.hi), str(k.lo)],
            "split": [[str(a.hi), str(a.lo)], [str(b.hi), str(b.lo)]],
            "fold": {str(i): [str(k.fold(i).hi), str(k.fold(i).lo)] for i in (0, 1, 2, 10, 1011, 2**40)},
            "uniform": fl(k.generator().random(70)),
            "normal": fl(k.generator().standard_normal(300)),
            "uniform_m2_2": fl(k.generator().uniform(-2.0, 2.0, 9)),
        }
        out["seeds"].append(rec)
    return out


def gen_hmc():
    """sampler.hmc_transition (sampler.py:163-203) on small models: chains of
    fixed-length HMC draws (accept/reject, stats) from fixed seeds."""
    out = []
    models = [std_normal_model(5), gaussian_model(np.logspace(-1, 1, 6)), funnel_model(4)]
    for mi, model in enumerate(models):
        for steps, eps in ((1, 0.3), (7, 0.25), (20, 0.9)):
            cfg = SamplerConfig(step_size=eps, mass=MassMatrix.identity(model.dim))
            q = np.linspace(-1.0, 1.2, model.dim)
            base = RngKey.from_seed(900 + 10 * mi + steps)
            draws = []
            for i in range(6):
                key = base.fold(i)
                q_new, st = tsampler.hmc_transition(q, cfg, model, key, steps)
                draws.append({"key": [str(key.hi), str(key.lo)], "q_in": fl(q), "q_out": fl(q_new),
                              "leapfrogs": st.leapfrog_calls, "diverged": bool(st.diverged),
                              "accept_stat": f(st.accept_stat), "energy": f(st.energy)})
                q = q_new
            out.append({"model": model_desc(model), "step": eps, "num_steps": steps, "draws": draws})
    return out


def main():
    only = sys.argv[1:]
    for name, fn in (("rng", gen_rng), ("trees", gen_trees), ("transitions", gen_transitions), ("runs", gen_runs),
                     ("logistic", gen_logistic), ("hmc", gen_hmc)):
        if only and name not in only:
            continue
        data = fn()
        with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
            json.dump(data, fh)
        print(name, "written")


if __name__ == "__main__":
    main()
