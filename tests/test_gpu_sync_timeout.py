"""Bounded waits of the persistent kernels.

Every inter-CTA / inter-GPU wait polls through a SpinGuard
(csrc/ts_logistic.cuh): past TS_SPIN_TIMEOUT_S the kernel gives up, raises
the model's sticky error word, and the host raises RuntimeError instead of
the GPU hanging.  TS_FAULT_INJECT=1 makes CTA 1 of the logistic grid never
arrive at the grid barrier - the single-GPU stand-in for a row-shard peer
that never launched.
"""

from __future__ import annotations

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _model(ts, seed=3):
    from tests_data import logistic_data

    x, y = logistic_data(20000, 54, seed)
    return ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision="fp32")


def test_missing_cta_times_out_instead_of_hanging(monkeypatch):
    import paper_1912_11554_b200 as ts

    monkeypatch.setenv("TS_SPIN_TIMEOUT_S", "0.2")
    monkeypatch.setenv("TS_FAULT_INJECT", "1")
    m = _model(ts)
    t0 = time.perf_counter()
    with pytest.raises(RuntimeError, match="synchronisation wait"):
        m.potential(np.zeros(55))
    # a run: every later wait gives up at once (sticky flag), so the whole
    # run ends quickly and every chain reports the timeout
    with pytest.raises(RuntimeError, match="synchronisation wait"):
        ts.run(ts.RunConfig(model={}, num_chains=1, num_warmup=20, num_samples=5, seed=1), m)
    assert time.perf_counter() - t0 < 60.0


def test_fresh_model_after_timeout_is_healthy(monkeypatch):
    import paper_1912_11554_b200 as ts

    monkeypatch.setenv("TS_SPIN_TIMEOUT_S", "0.2")
    monkeypatch.setenv("TS_FAULT_INJECT", "1")
    bad = _model(ts)
    with pytest.raises(RuntimeError):
        bad.potential(np.zeros(55))
    monkeypatch.delenv("TS_FAULT_INJECT")
    good = _model(ts)
    u = good.potential(np.zeros(55))
    assert np.isclose(u, 20000 * np.log(2.0), rtol=1e-6)
    res = ts.run(ts.RunConfig(model={}, num_chains=1, num_warmup=20, num_samples=5, seed=1), good)
    assert np.isfinite(res[0].samples).all()
