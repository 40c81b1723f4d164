"""Posterior moments of eight schools (non-centred) from the REFERENCE sampler.

Usage (from the repo root, where /root/reference exists):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_eight_schools_moments.py

The reference has no eight-schools built-in; its plugin API takes any
TargetModel (models.py:25-40), so the model is the oracle twin
(oracle/turnstile_oracle.py eight_schools_potential/gradient, the same
density as csrc/ts_models.cuh) run through the unmodified reference
``chains.run_chain`` (chains.py:98-163) - one process per chain, all host
cores (chains are independent and prefix-stable, tests/test_chains.py:70-72).
Writes tests/golden/eight_schools_moments.json: pooled mean / SD, the
reference estimator's ESS (diagnostics.py:49-86) and split R-hat
(diagnostics.py:89-105) per dimension, and MCSEs.  Seed 11 and 64 chains:
statistically independent of the device test's chains (seed 3).
"""

from __future__ import annotations

import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
SEED, CHAINS, W, S = 11, 64, 1000, 1000


def _setup():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")


def _chain(c):
    _setup()
    from turnstile import chains as tchains
    from turnstile.models import TargetModel
    from turnstile_oracle import eight_schools_gradient, eight_schools_potential

    y = [28.0, 8.0, -3.0, 7.0, -1.0, 1.0, 18.0, 12.0]
    s = [15.0, 10.0, 16.0, 11.0, 9.0, 11.0, 10.0, 18.0]
    model = TargetModel("eight_schools", 10, lambda q: eight_schools_potential(q, y, s),
                        lambda q: eight_schools_gradient(q, y, s), {"y": y, "sigma": s})
    cfg = tchains.RunConfig(model={"model": "eight_schools"}, num_chains=CHAINS, num_warmup=W, num_samples=S, seed=SEED)
    key = tchains.chain_keys(SEED, CHAINS)[c]
    r = tchains.run_chain(c, key, model, cfg, tchains._base_config(cfg, model))
    return r.samples, r.total_leapfrogs, r.divergences


def main():
    _setup()
    from turnstile import diagnostics

    t0 = time.time()
    with Pool(os.cpu_count()) as pool:
        out = pool.map(_chain, range(CHAINS))
    chains = np.stack([o[0] for o in out])
    pooled = chains.reshape(-1, chains.shape[-1])
    mean, sd = pooled.mean(0), pooled.std(0, ddof=1)
    ess = diagnostics.ess(chains)
    rhat = diagnostics.split_rhat(chains)
    rec = {
        "generator": "reference turnstile.chains.run_chain + eight-schools TargetModel twin (oracle)",
        "seed": SEED, "num_chains": CHAINS, "num_warmup": W, "num_samples": S,
        "mean": mean.tolist(), "sd": sd.tolist(), "ess": ess.tolist(), "split_rhat": rhat.tolist(),
        "mcse_mean": (sd / np.sqrt(ess)).tolist(), "mcse_sd": (sd / np.sqrt(2.0 * ess)).tolist(),
        "total_leapfrogs": int(sum(o[1] for o in out)), "divergences": int(sum(o[2] for o in out)),
        "cpu_seconds_wall": time.time() - t0, "cores": os.cpu_count(),
    }
    with open(os.path.join(HERE, "eight_schools_moments.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps({k: v for k, v in rec.items() if not isinstance(v, list)}))


if __name__ == "__main__":
    main()
