"""Synthetic data generators shared by tests, bench.py and tests/golden/make_golden.py.

Data rule: generate in fp64 with numpy.random.default_rng(seed),
round X to fp32, and feed the identical values to the reference/oracle
(as fp64) and to the device (as fp32).
"""

from __future__ import annotations

import numpy as np


def logistic_data(n: int, p: int, seed: int):
    """X ~ N(0,1) rounded to fp32; w* ~ N(0, 1/p), b* = 0; y ~ Bernoulli(sigmoid(X w*))."""
    g = np.random.default_rng(seed)
    x = g.standard_normal((n, p)).astype(np.float32).astype(np.float64)
    w = g.standard_normal(p) / np.sqrt(p)
    y = (g.random(n) < 1.0 / (1.0 + np.exp(-(x @ w)))).astype(np.float64)
    return x, y
