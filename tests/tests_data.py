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


def logistic_data_f32(n: int, p: int, seed: int, chunk_rows: int = 1 << 18, rows=None):
    """The same values as logistic_data(n, p, seed), produced in row chunks so
    large shapes (config 5: 8M x 255) never hold an fp64 copy of X.  Returns
    (X fp32, y uint8) for rows [a, b) = `rows` (default all).  The generator's
    normal stream is consumed in C order, so chunking rows reproduces the
    one-shot draw exactly; rows outside [a, b) are drawn and dropped."""
    a, b = (0, n) if rows is None else rows
    g = np.random.default_rng(seed)
    x = np.empty((b - a, p), dtype=np.float32)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        if r1 <= a or r0 >= b:
            g.standard_normal((r1 - r0, p))
            continue
        blk = g.standard_normal((r1 - r0, p))
        lo, hi = max(a, r0), min(b, r1)
        x[lo - a:hi - a] = blk[lo - r0:hi - r0]
    w = g.standard_normal(p) / np.sqrt(p)
    eta = np.empty(b - a, dtype=np.float64)
    for r0 in range(0, b - a, chunk_rows):
        r1 = min(b - a, r0 + chunk_rows)
        eta[r0:r1] = x[r0:r1].astype(np.float64) @ w
    u = g.random(n)[a:b]
    y = (u < 1.0 / (1.0 + np.exp(-eta))).astype(np.uint8)
    return x, y
