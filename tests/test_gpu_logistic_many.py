"""Many chains sharing X on the tcgen05 tensor cores (logistic precision
"tf32", csrc/ts_k_logistic_many.cu) - BASELINE north star "many-chain
batching" / VERDICT r1 row N3.

Stated tolerance of the policy (eta in 3xTF32, gradient in 3xBF16, fp32
accumulation in TMEM): U within 1e-6 relative + 1e-3 absolute nats,
gradient within 2e-5 relative of max |g| + 1e-2 absolute, against the fp64
oracle (kernels.py:90-123 restated).  Its acceptance
decisions are checked against the FP32 and FP64 policies by replaying
transitions from the same states (flips counted, each at a near-tie).
Chains are independent of the batch they share a step with: a chain run
alone reproduces its batched run bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U_REL, U_ABS = 1e-6, 1e-3
G_REL, G_ABS = 2e-5, 1e-2


def _ts():
    import paper_1912_11554_b200 as t

    return t


@pytest.mark.parametrize("n,p,seed", [(3000, 54, 11), (777, 10, 12), (129, 62, 13), (1, 3, 14), (581012, 54, 20191222)])
def test_logistic_many_potential_gradient(n, p, seed, oracle):
    from tests_data import logistic_data

    t = _ts()
    x, y = logistic_data(n, p, seed)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="tf32")
    om = oracle.Model("logistic_regression", p + 1, x=x, y=y, fused_omp=True)
    rng = np.random.default_rng(seed)
    for q in (np.zeros(p + 1), rng.standard_normal(p + 1) * 0.1, rng.standard_normal(p + 1)):
        got = t.models.potential_and_gradient(m.device_spec, q[None, :])[0]
        U, g = om._fused(q.tolist())
        g = np.asarray(g)
        print(f"tf32 many n={n} p={p}: |dU| {abs(got[0] - U):.3e} (U {U:.4g}), max|dg| "
              f"{np.abs(got[1:] - g).max():.3e} (max|g| {np.abs(g).max():.4g})")
        assert abs(got[0] - U) <= U_REL * abs(U) + U_ABS, (got[0], U)
        assert np.abs(got[1:] - g).max() <= G_REL * np.abs(g).max() + G_ABS, np.abs(got[1:] - g).max()


def test_logistic_many_chains_independent_of_batch():
    """A chain's draws do not depend on which other chains share its steps."""
    from tests_data import logistic_data

    t = _ts()
    x, y = logistic_data(20000, 54, 5)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="tf32")
    cfg = t.RunConfig(model={}, num_chains=64, num_warmup=40, num_samples=20, seed=9)
    keys = t.chain_keys(9, 64)
    big = t.run_device(m, cfg, keys, 0)
    s_big = big.samples.cpu().numpy()
    st_big = big.stats.cpu().numpy()
    assert (big.status.cpu().numpy() == 0).all()
    for c in (0, 5, 63):
        one = t.run_device(m, cfg, [keys[c]], 0)
        assert np.array_equal(one.samples.cpu().numpy()[0], s_big[c]), c
        assert np.array_equal(one.stats.cpu().numpy()[0], st_big[c]), c


def test_logistic_many_decisions_vs_fp32_and_fp64(oracle):
    """Replay transitions of an fp64 run from the same states with the tf32
    many-chain policy, the fp32 policy and the fp64 policy: integer decisions
    compared, flips counted (bound: 4 of 64 at this size) and each flip's
    smallest oracle decision margin <= 1e-3 (a near-tie)."""
    from tests_data import logistic_data

    t = _ts()
    x, y = logistic_data(50000, 54, 21)
    models = {p: t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=p) for p in ("tf32", "fp32", "fp64")}
    W, S, seed = 150, 64, 31
    key = t.chain_keys(seed, 1)[0]
    r = t.run_device(models["fp64"], t.RunConfig(model={}, num_chains=1, num_warmup=W, num_samples=S, seed=seed), [key], 0)
    ad = r.adapt.cpu().numpy()[0]
    samples = r.samples.cpu().numpy()[0]
    scfg = t.SamplerConfig(step_size=float(ad[1]), mass=t.MassMatrix(ad[2 + W:].copy()))
    om = oracle.Model("logistic_regression", 55, x=x, y=y, fused_omp=True)
    flips = {"tf32": [], "fp32": []}
    for i in range(1, S):
        q0 = samples[i - 1]
        dkey = key.fold(10 + W + i)
        dec = {}
        for prec, m in models.items():
            ug = t.models.potential_and_gradient(m.device_spec, q0[None, :])[0]
            z = t.PhasePoint(q0, np.zeros(55), float(ug[0]), ug[1:].copy())
            _, st, tr = t.nuts_transition_from(z, scfg, m, dkey, return_trace=True)
            dec[prec] = (st.depth_reached, st.leapfrog_calls, int(st.diverged),
                         tuple((j, gr, c, stp) for j, c, stp, gr, _ in tr.trees), (tr.proposal_tree, tr.proposal_leaf))
        for prec in ("tf32", "fp32"):
            if dec[prec] != dec["fp64"]:
                U0, g0 = om._fused(q0.tolist())
                margins = []
                oracle.transition(oracle.Point(q0.tolist(), [0.0] * 55, U0, list(g0)), scfg.step_size,
                                  scfg.mass.inv_diag.tolist(), om, (dkey.hi, dkey.lo), margins=margins)
                mrg = min((mm for tm in margins for mm in tm), key=lambda km: km[1], default=("none", np.inf))
                flips[prec].append((i, mrg))
    print("decision flips vs fp64 over", S - 1, "transitions:", {k: len(v) for k, v in flips.items()}, flips)
    for prec in ("tf32", "fp32"):
        assert len(flips[prec]) <= 4, flips
        assert all(m[1] <= 1e-3 for _, m in flips[prec]), flips


def test_logistic_many_posterior_matches_fp64():
    """64 tf32 chains vs 4 fp64 chains on a 20k-row model: means and SDs
    within 4 MCSE, R-hat < 1.01."""
    from tests_data import logistic_data

    t = _ts()
    x, y = logistic_data(20000, 54, 8)
    res = {}
    for prec, C in (("tf32", 64), ("fp64", 4)):
        m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=prec)
        r = t.run(t.RunConfig(model={}, num_chains=C, num_warmup=500, num_samples=500, seed=4), m)
        res[prec] = np.stack([c.samples for c in r])
    out = {}
    for prec, ch in res.items():
        pooled = ch.reshape(-1, 55)
        mu = pooled.mean(0)
        # the SD's Monte-Carlo error uses the ESS of the squared deviations:
        # NUTS draws are antithetic for the mean (ESS above the draw count),
        # not for second moments
        out[prec] = (mu, pooled.std(0, ddof=1), t.ess(ch), t.ess((ch - mu) ** 2), t.split_rhat(ch))
    (m1, s1, e1, q1, r1), (m2, s2, e2, q2, r2) = out["tf32"], out["fp64"]
    assert (r1 < 1.01).all() and (r2 < 1.01).all()
    z = np.abs(m1 - m2) / np.sqrt(s1 ** 2 / e1 + s2 ** 2 / e2)
    zs = np.abs(s1 - s2) / np.sqrt(s1 ** 2 / (2 * q1) + s2 ** 2 / (2 * q2))
    print(f"tf32 many-chain vs fp64: max z(mean) {z.max():.2f}, max z(sd) {zs.max():.2f}")
    assert (z < 4).all() and (zs < 4).all()
