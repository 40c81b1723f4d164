"""The reference's sampler/run/acceptance battery, executed on the device.

Follows reference tests/test_sampler.py:43-208, tests/test_chains.py:76-131
and tests/test_acceptance.py:125-136 (criterion 6) case by case: the same
models, seeds, step sizes and thresholds, with every draw produced by the
persistent device run (``run``) instead of the CPU sampler.  Per-transition
loops of the reference (``nuts_transition`` in a Python loop) are expressed
as one device run with ``num_warmup=0`` and a fixed step size - the same
Markov chain, one launch.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DESCRIPTORS = [
    {"model": "std_normal", "params": {"dim": 2}},
    {"model": "gaussian", "params": {"cov_diag": [2.0, 0.5]}},
    {"model": "funnel", "params": {"dim": 3}},
]


def t():
    import paper_1912_11554_b200 as ts

    return ts


def small(desc, mode="sequential", seed=7, **kw):
    kw.setdefault("num_chains", 4)
    return t().RunConfig(model=desc, num_warmup=25, num_samples=25, mode=mode, seed=seed, **kw)


def fixed(desc, step, samples, seed, chains=1, **sampler_kw):
    ts = t()
    dim = ts.model_from_descriptor(desc).dim
    base = ts.SamplerConfig(step_size=step, mass=ts.MassMatrix.identity(dim), **sampler_kw)
    return ts.RunConfig(model=desc, num_chains=chains, num_warmup=0, num_samples=samples, seed=seed, sampler=base)


def test_depth_cap_one_is_single_step_accept_reject():
    """test_sampler.py:44-56."""
    res = t().run(fixed({"model": "std_normal", "params": {"dim": 1}}, 0.9, 4000, 1, max_tree_depth=1))[0]
    assert (res.stats_array[:, 1] == 1).all()
    draws = res.samples[500:, 0]
    assert abs(draws.mean()) < 0.1
    assert 0.8 < draws.var() < 1.2


def test_periodic_target_terminates_before_depth_cap():
    """test_sampler.py:58-67."""
    res = t().run(fixed({"model": "std_normal", "params": {"dim": 1}}, 0.1, 1000, 7))[0]
    assert (res.stats_array[:, 0] < 10).sum() >= 990


def test_accept_stat_in_unit_interval_and_energy_finite():
    """test_sampler.py:97-106."""
    res = t().run(fixed({"model": "std_normal", "params": {"dim": 2}}, 0.5, 100, 9))[0]
    st = res.stats_array
    assert ((st[:, 3] >= 0.0) & (st[:, 3] <= 1.0)).all()
    assert np.isfinite(st[:, 4]).all() and (st[:, 1] >= 1).all()


def test_divergence_recorded_not_raised():
    """test_sampler.py:108-119: a huge step diverges, the chain stays finite."""
    res = t().run(fixed({"model": "std_normal", "params": {"dim": 1}}, 50.0, 50, 3, divergence_threshold=50.0))[0]
    assert res.divergences > 0
    assert np.isfinite(res.samples).all()


def test_funnel_divergences_at_large_step():
    """The funnel's neck diverges at a fixed large step (divergence workload)."""
    res = t().run(fixed({"model": "funnel", "params": {"dim": 10}}, 1.0, 400, 5, chains=4))
    assert sum(r.divergences for r in res) > 0
    assert all(np.isfinite(r.samples).all() for r in res)


@pytest.mark.parametrize("dim", [1, 5])
def test_ks_against_exact_marginals(dim):
    """test_sampler.py:174-188."""
    from scipy import stats

    cfg = t().RunConfig(model={"model": "std_normal", "params": {"dim": dim}}, num_chains=4, num_warmup=200,
                        num_samples=5000, seed=60 + dim)
    pooled = np.concatenate([r.samples for r in t().run(cfg)])
    for d in range(dim):
        assert stats.kstest(pooled[:, d], "norm").pvalue > 0.001 / dim


def test_classic_ks_against_exact_marginals():
    """test_sampler.py:191-208: the classic criterion end to end."""
    from scipy import stats

    ts = t()
    base = ts.SamplerConfig(step_size=1.0, mass=ts.MassMatrix.identity(2), criterion="classic")
    cfg = ts.RunConfig(model={"model": "std_normal", "params": {"dim": 2}}, num_chains=4, num_warmup=200,
                       num_samples=3000, seed=71, sampler=base)
    pooled = np.concatenate([r.samples for r in ts.run(cfg)])
    for d in range(2):
        assert stats.kstest(pooled[:, d], "norm").pvalue > 0.001 / 2


def test_criterion_6_warmup_adaptation():
    """test_acceptance.py:125-136: inverse mass within 2x, mean accept in [0.7, 0.9]."""
    cfg = t().RunConfig(model={"model": "gaussian", "params": {"cov_diag": [100.0, 0.01]}}, num_chains=2,
                        num_warmup=1000, num_samples=500, seed=11)
    res = t().run(cfg)
    truth = np.array([100.0, 0.01])
    for r in res:
        ratio = np.array(r.adaptation["inv_mass_diag"]) / truth
        assert ((ratio >= 0.5) & (ratio <= 2.0)).all(), ratio
    accept = float(np.mean(np.concatenate([r.stats_array[:, 3] for r in res])))
    assert 0.7 <= accept <= 0.9, accept


@pytest.mark.parametrize("desc", DESCRIPTORS, ids=lambda d: d["model"])
def test_mode_invariance_bitwise(desc):
    """test_chains.py:76-84."""
    seq = t().run(small(desc, "sequential"))
    par = t().run(small(desc, "parallel"))
    for a, b in zip(seq, par, strict=True):
        assert np.array_equal(a.samples, b.samples)
        assert np.array_equal(a.stats_array, b.stats_array)
        assert a.adaptation["final_step_size"] == b.adaptation["final_step_size"]


def test_reproducible_distinct_chains_and_seeds():
    """test_chains.py:86-108."""
    desc = DESCRIPTORS[0]
    a, b = t().run(small(desc)), t().run(small(desc))
    for r1, r2 in zip(a, b):
        assert np.array_equal(r1.samples, r2.samples)
    assert len({tuple(r.samples[:, 0]) for r in a}) == len(a)
    assert not np.array_equal(t().run(small(desc, seed=1))[0].samples, t().run(small(desc, seed=2))[0].samples)


def test_chain_prefix_stability_on_device():
    """Adding chains does not change existing chains (test_chains.py:70-72, end to end)."""
    desc = DESCRIPTORS[1]
    two = t().run(small(desc, num_chains=2))
    six = t().run(small(desc, num_chains=6))
    for r1, r2 in zip(two, six[:2]):
        assert np.array_equal(r1.samples, r2.samples)


def test_leapfrog_totals_consistent():
    """test_chains.py:118-123."""
    for r in t().run(small(DESCRIPTORS[0])):
        assert r.sampling_leapfrogs == sum(s.leapfrog_calls for s in r.stats)
        assert r.total_leapfrogs >= r.sampling_leapfrogs
        assert r.samples.shape == (25, 2)


def test_zero_warmup_uses_fixed_settings():
    """test_chains.py:125-130."""
    res = t().run(fixed(DESCRIPTORS[0], 0.7, 10, 3))
    assert res[0].adaptation["final_step_size"] == 0.7
