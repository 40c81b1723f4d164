"""North-star parity layer 3 on BASELINE configs: posterior moments within
Monte-Carlo error of the reference, R-hat < 1.01 (reference criteria:
tests/test_acceptance.py:100-136, estimators diagnostics.py:49-105).

Eight schools (config 3): the device's 8192-chain run (seed 3) against the
reference sampler's own moments (64 independent chains, seed 11, plugin
twin of the model) committed by tests/golden/make_eight_schools_moments.py.
Covtype (config 2) is in test_gpu_covtype_fp32.py (fp32 vs fp64 policies).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_eight_schools_8192_chains_match_reference_moments():
    import paper_1912_11554_b200 as ts

    ref = golden("eight_schools_moments")
    C, W, S = 8192, 1000, 1000
    model = ts.eight_schools_model()
    cfg = ts.RunConfig(model={"model": "eight_schools"}, num_chains=C, num_warmup=W, num_samples=S, seed=3)
    r = ts.run_device(model, cfg, ts.chain_keys(3, C), 0)
    x = r.samples  # (C, S, D) on the device
    mean = x.mean(dim=(0, 1)).cpu().numpy()
    sd = x.reshape(-1, x.shape[-1]).std(dim=0, unbiased=True).cpu().numpy()
    ess = ts.ess_device(x)
    rhat = ts.split_rhat_device(x)
    assert (rhat < 1.01).all(), rhat
    mcse_mean = np.sqrt(sd ** 2 / ess + np.asarray(ref["mcse_mean"]) ** 2)
    mcse_sd = np.sqrt(sd ** 2 / (2 * ess) + np.asarray(ref["mcse_sd"]) ** 2)
    z_mean = np.abs(mean - np.asarray(ref["mean"])) / mcse_mean
    z_sd = np.abs(sd - np.asarray(ref["sd"])) / mcse_sd
    print(f"eight schools vs reference: max |dmean|/MCSE {z_mean.max():.2f}, max |dsd|/MCSE {z_sd.max():.2f}, "
          f"min device ESS {ess.min():.0f}, max R-hat {rhat.max():.4f}")
    assert (z_mean < 4.0).all(), z_mean
    assert (z_sd < 4.0).all(), z_sd
