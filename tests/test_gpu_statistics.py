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


def test_dense_config4_moments_tf32():
    """North-star layer 3 at BASELINE config 4 (1000-D correlated Gaussian,
    dense mass M^-1 = Sigma, 1024 chains, the tcgen05 TF32 path): every
    coordinate's posterior mean and variance against the exact target
    (mean 0, Sigma = Q diag(logspace(-2, 2)) Q^T) within Monte-Carlo error,
    split R-hat < 1.01 -- the TF32 gradients do not bias the sampler."""
    import torch

    import paper_1912_11554_b200 as t

    D, C, W, S = 1000, 1024, 150, 150
    g = np.random.default_rng(4)
    Q, _ = np.linalg.qr(g.standard_normal((D, D)))
    lam = np.logspace(-2, 2, D)
    Sigma = (Q * lam) @ Q.T
    P = (Q / lam) @ Q.T
    m = t.dense_gaussian_model(P, inv_mass=Sigma, precision="tf32")
    cfg = t.RunConfig(model={}, num_chains=C, num_warmup=W, num_samples=S, seed=4)
    r = t.run_device(m, cfg, t.chain_keys(4, C), 0)
    x = r.samples  # (C, S, D) on the device, q-space
    ess, rhat = t.chain_diagnostics_device(x)
    assert np.nanmax(rhat) < 1.01, np.nanmax(rhat)
    flat = x.reshape(-1, D)
    mean = flat.mean(0).cpu().numpy()
    var = flat.var(0).cpu().numpy()
    sd = np.sqrt(np.diag(Sigma))
    mcse_mean = sd / np.sqrt(ess)
    z_mean = np.abs(mean) / mcse_mean
    # variance: MCSE from the ESS of the squared deviations (NUTS draws are
    # antithetic for the mean -- ESS above the draw count -- not for squares);
    # for a Gaussian marginal sd((x - mu)^2) = sqrt(2) var
    ess_sq, _ = t.chain_diagnostics_device((x - torch.from_numpy(mean).to(x.device)) ** 2)
    z_var = np.abs(var - np.diag(Sigma)) / (np.diag(Sigma) * np.sqrt(2.0 / ess_sq))
    print(f"config 4 tf32: max |mean|/MCSE {z_mean.max():.2f}, max |dvar|/MCSE {z_var.max():.2f}, "
          f"min ESS {np.nanmin(ess):.0f} (squares {np.nanmin(ess_sq):.0f}), max R-hat {np.nanmax(rhat):.4f}")
    # 1000 coordinates: a 5-sigma bound keeps the family-wise false alarm rate ~6e-4
    assert z_mean.max() < 5.0, z_mean.max()
    assert z_var.max() < 5.0, z_var.max()
