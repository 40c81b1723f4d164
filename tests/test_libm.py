"""The device's exp / log1p / log (csrc/ts_libm.cuh) against this image's
glibc, which the reference calls through Python's math module.  The header
is compiled for the host with g++ (no FMA contraction: only its explicit
fma() calls) and evaluated on random inputs over the ranges the sampler uses
(Metropolis terms exp(-dH), log-sum-exp arguments in [0, 1], dual averaging)
plus wide and special values; exp and log1p must be bitwise equal, log
equal except where glibc itself is not correctly rounded (rate measured)."""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import tempfile

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def probe():
    d = tempfile.mkdtemp(prefix="ts_libm_")
    so = os.path.join(d, "libm_probe.so")
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                           os.path.join(HERE, "libm_probe.cpp")])
    lib = ctypes.CDLL(so)
    for f in ("probe_exp", "probe_log1p", "probe_log"):
        getattr(lib, f).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]
    return lib


def _run(lib, fn, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    getattr(lib, fn)(x.ctypes.data, y.ctypes.data, x.size)
    return y


def _glibc(f, x):
    """math.<f> elementwise (glibc); domain / range errors mapped to the libm value."""
    out = []
    for v in x.tolist():
        try:
            out.append(f(v) if not math.isnan(v) else math.nan)
        except OverflowError:
            out.append(math.inf)
        except ValueError:  # log1p(-1), log(0): -inf; below the domain: nan
            out.append(-math.inf if v in (-1.0, 0.0) and f is not math.exp else math.nan)
    return np.array(out)


def _inputs_exp(rng, n):
    return np.concatenate([
        -rng.exponential(3.0, n),                 # exp(-dH), dH > 0
        rng.uniform(-40.0, 40.0, n),
        rng.uniform(-745.0, 709.0, n // 4),       # incl. the subnormal / overflow special cases
        rng.uniform(-1.0, 1.0, n // 4) * 2.0 ** -rng.integers(0, 60, n // 4),
        np.array([0.0, -0.0, 1.0, -1.0, 709.78, -745.2, -1000.0, 1000.0, math.inf, -math.inf]),
    ])


def _inputs_log1p(rng, n):
    return np.concatenate([
        rng.uniform(0.0, 1.0, n),                  # log1p(exp(lo - hi)) in the log-sum-exp
        np.exp(rng.uniform(-745.0, 0.0, n // 2)),
        rng.uniform(-0.9999, 10.0, n // 2),
        -np.exp(rng.uniform(-60.0, 0.0, n // 4)),
        np.exp(rng.uniform(-30.0, 700.0, n // 4)),
        np.array([0.0, -0.0, -1.0, 1.0, 0.41421, -0.29289, 2.0 ** -29, 2.0 ** -54, math.inf]),
    ])


def test_exp_matches_glibc_bitwise(probe):
    x = _inputs_exp(np.random.default_rng(1), 400_000)
    got = _run(probe, "probe_exp", x)
    ref = _glibc(math.exp, x)
    same = (got.view(np.uint64) == ref.view(np.uint64))
    assert same.all(), (x[~same][:5], got[~same][:5], ref[~same][:5])


def test_log1p_matches_glibc_bitwise(probe):
    x = _inputs_log1p(np.random.default_rng(2), 400_000)
    got = _run(probe, "probe_log1p", x)
    ref = _glibc(math.log1p, x)
    same = (got.view(np.uint64) == ref.view(np.uint64))
    assert same.all(), (x[~same][:5], got[~same][:5], ref[~same][:5])


def test_log_correctly_rounded_and_glibc_on_dual_averaging_inputs(probe):
    rng = np.random.default_rng(3)
    # dual averaging starts from mu = log(10 eps0), log(eps0), eps0 = 2^k x base step
    k = np.arange(-60, 61, dtype=np.float64)
    da = np.concatenate([2.0 ** k, 10.0 * 2.0 ** k])
    got = _run(probe, "probe_log", da)
    ref = _glibc(math.log, da)
    assert (got.view(np.uint64) == ref.view(np.uint64)).all()
    # random inputs: equal to glibc except where glibc misrounds (~1e-4)
    x = np.concatenate([np.exp(rng.uniform(-700, 700, 200_000)), rng.uniform(0.5, 2.0, 200_000)])
    got = _run(probe, "probe_log", x)
    ref = _glibc(math.log, x)
    mis = np.nonzero(got.view(np.uint64) != ref.view(np.uint64))[0]
    rate = mis.size / x.size
    assert rate < 2e-3, rate  # measured 7.5e-4: glibc's log is not correctly rounded there
    assert np.all(np.abs(got - ref) <= np.spacing(np.abs(ref)))
    # ... and where they differ, ours is the correctly rounded value
    from decimal import Decimal, getcontext

    getcontext().prec = 60
    for i in mis[:200]:
        assert float(Decimal(float(x[i])).ln()) == got[i], x[i]
