"""Host-side logic of the package (no GPU): API validation, schedule,
adaptation recursions, diagnostics, and the C ABI library's exports.

KATs are the reference's own (file:line under /root/reference/pkg/tests).
"""

from __future__ import annotations

import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1912_11554_b200 as t
from conftest import ROOT, golden, nums

# ----------------------------------------------------------------------------- C ABI


def _lib_path():
    path = os.path.join(ROOT, "paper_1912_11554_b200", "libturnstile_b200.so")
    if not os.path.exists(path):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "paper_1912_11554_b200", "csrc"), "-j4"])
    return path


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "turnstile_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(ts_\w+)\(", header, flags=re.M))
    assert declared >= {"ts_model_create", "ts_build_tree", "ts_transition", "ts_run_chains", "ts_potential_grad"}
    lib = ctypes.CDLL(_lib_path())
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(t._lib.EXPORTS) == declared


def test_library_abi_version_and_error_path():
    lib = t._lib.load_library(_lib_path())
    assert lib.ts_abi_version() == t._lib.ABI_VERSION
    out = t._lib._P()
    code = lib.ts_model_create(99, 3, None, 0, None, None, 0, 0, 0, ctypes.byref(out))
    assert code == t._lib.TS_EINVAL
    assert b"unknown model kind" in lib.ts_last_error()
    with pytest.raises(ValueError):
        t._lib.check(code)


def test_no_cpu_fallback_without_cuda(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    m = t.std_normal_model(3)
    with pytest.raises(RuntimeError, match="CUDA device"):
        m.potential(np.zeros(3))


def test_callable_models_are_rejected():
    m = t.TargetModel("custom", 2, lambda q: 0.0, lambda q: q)
    cfg = t.SamplerConfig(step_size=0.1, mass=t.MassMatrix.identity(2))
    z = t.PhasePoint(np.zeros(2), np.zeros(2), 0.0, np.zeros(2))
    with pytest.raises(ValueError, match="no device implementation"):
        t.build_tree_iterative(z, 2, 0.1, cfg, m, t.RngKey.from_seed(0))
    with pytest.raises(ValueError):
        t.run(t.RunConfig(model={}, num_chains=1, num_warmup=0, num_samples=4), m)


# ----------------------------------------------------------------------------- treemath (test_treemath.py:301-401)


def test_bit_kats():
    assert t.bit_count(6) == 2 and t.bit_count(11) == 3
    assert t.trailing_ones(11) == 2 and t.trailing_ones(7) == 3 and t.trailing_ones(6) == 0
    assert t.candidate_set(11) == [(10, 2), (8, 1)]
    assert t.candidate_set(7) == [(6, 2), (4, 1), (0, 0)]
    assert t.candidate_set(6) == []


def test_candidate_sets_brute_force():
    for n in range(1 << 14):
        expect = [(t.subtree_leftmost(n, k), t.bit_count(t.subtree_leftmost(n, k)))
                  for k in range(1, t.trailing_ones(n) + 1)]
        assert t.candidate_set(n) == expect
        if n:
            # i_max = popcount(n - 1)-style identity used by the device schedule
            if n % 2 == 1:
                assert t.bit_count(n) - 1 == t.bit_count(n - 1)


# ----------------------------------------------------------------------------- config validation


def test_sampler_config_validation():
    mass = t.MassMatrix.identity(2)
    for kw in ({"step_size": 0.0}, {"step_size": math.inf}, {"max_tree_depth": 0}, {"max_tree_depth": 31},
               {"criterion": "sideways"}, {"tree_builder": "magic"}, {"divergence_threshold": 0.0}):
        args = {"step_size": 0.1, "mass": mass, **kw}
        with pytest.raises(ValueError):
            t.SamplerConfig(**args)


def test_run_config_validation():
    for kw in ({"num_chains": 0}, {"num_samples": 0}, {"num_warmup": 5}, {"mode": "turbo"}):
        with pytest.raises(ValueError):
            t.RunConfig(model={}, **kw)


def test_mass_matrix_validation():
    with pytest.raises(ValueError):
        t.MassMatrix([1.0, -1.0])
    with pytest.raises(ValueError):
        t.MassMatrix([])
    assert np.allclose(t.MassMatrix([4.0]).momentum_std, [0.5])


def test_depth_validation_host_side():
    m = t.std_normal_model(1)
    cfg = t.SamplerConfig(step_size=0.1, mass=t.MassMatrix.identity(1), max_tree_depth=12)
    z = t.PhasePoint(np.zeros(1), np.ones(1), 0.0, np.zeros(1))
    for depth in (-1, 13):
        with pytest.raises(ValueError):
            t.build_tree_iterative(z, depth, 0.1, cfg, m, t.RngKey.from_seed(0))


# ----------------------------------------------------------------------------- adaptation (test_adapt.py)


def test_dual_averaging_one_step_kat():
    s = t.DualAveragingState.init(1.0)
    s = t.da_update(s, 0.0)
    assert s.h_bar == pytest.approx(0.8 / 11)
    assert s.log_eps == pytest.approx(math.log(10.0) - 1.0 / 0.05 * 0.8 / 11)


def test_warmup_schedule_goldens():
    s = t.warmup_schedule(1000)
    assert s.phases == (("init", 150), ("window", 25), ("window", 50), ("window", 100), ("window", 200),
                        ("window", 300), ("window", 75), ("terminal", 100))
    inside, ends = s.window_steps()
    assert ends == {174, 224, 324, 524, 824, 899}
    flags = s.device_flags()
    assert set(np.nonzero(flags & 2)[0].tolist()) == ends
    assert set(np.nonzero(flags & 1)[0].tolist()) == inside
    with pytest.raises(ValueError):
        t.warmup_schedule(19)


def test_schedule_matches_oracle(oracle):
    for W in (20, 37, 100, 150, 1000, 2500):
        assert t.warmup_schedule(W).device_flags().tolist() == oracle.schedule_flags(W)


def test_da_weights_are_python_pow():
    w = t.adapt.da_weights(50)
    assert w.tolist() == [k ** (-0.75) for k in range(1, 51)]


def test_welford_and_regularized_variance():
    rng = np.random.default_rng(0)
    xs = rng.standard_normal((50, 3))
    st = t.WelfordState.init(3)
    for x in xs:
        st = t.welford_update(st, x)
    assert np.allclose(t.welford_variance(st), xs.var(axis=0, ddof=1))
    reg = t.welford_regularized_variance(st)
    assert np.allclose(reg, (50 / 55) * xs.var(axis=0, ddof=1) + (5 / 55) * 1e-3)


# ----------------------------------------------------------------------------- rng


def test_rng_keys_match_golden():
    for rec in golden("rng")["seeds"]:
        k = t.RngKey.from_seed(int(rec["seed"]))
        assert [str(k.hi), str(k.lo)] == rec["key"]
        assert [str(k.fold(10).hi), str(k.fold(10).lo)] == rec["fold"]["10"]


def test_chain_keys_prefix_stable():
    a = t.chain_keys(5, 3)
    b = t.chain_keys(5, 8)
    assert a == b[:3] and len(set(b)) == 8


# ----------------------------------------------------------------------------- diagnostics


def test_ess_and_rhat_match_oracle(oracle):
    rng = np.random.default_rng(1)
    chains = np.cumsum(rng.standard_normal((4, 400, 3)) * 0.3, axis=1) * 0.1 + rng.standard_normal((4, 400, 3))
    assert np.allclose(t.ess(chains), oracle.ess(chains))
    r = t.split_rhat(chains)
    assert r.shape == (3,) and np.all(r > 0.99)


def test_ess_iid_close_to_draw_count():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((4, 1000, 2))
    e = t.ess(x)
    assert (e > 3000).all() and (e <= 4000).all()


def test_constant_dimension_warns():
    x = np.zeros((2, 20, 1))
    with pytest.warns(RuntimeWarning):
        assert math.isnan(t.ess(x)[0])


# ----------------------------------------------------------------------------- data / descriptors


def test_logistic_data_validation():
    with pytest.raises(ValueError):
        t.LogisticRegressionData(np.zeros((3, 2)), np.zeros(2))
    with pytest.raises(ValueError):
        t.LogisticRegressionData(np.zeros((2, 2)), np.array([0.0, 2.0]))
    with pytest.raises(ValueError):
        t.LogisticRegressionData(np.array([[np.nan, 0.0]]), np.array([1.0]))


def test_model_from_descriptor_and_csv(tmp_path):
    m = t.model_from_descriptor({"model": "gaussian", "params": {"cov_diag": [1.0, 4.0]}})
    assert m.dim == 2 and np.allclose(m.device_spec.params, [1.0, 0.25])
    csv = tmp_path / "d.csv"
    csv.write_text("a,b,label\n0.5,1.0,1\n-1.0,2.0,0\n")
    (tmp_path / "m.json").write_text('{"model": "logistic_regression", "data_path": "d.csv"}')
    m = t.model_from_descriptor(str(tmp_path / "m.json"))
    assert m.dim == 3 and m.device_spec.x.dtype == np.float32 and m.device_spec.y.tolist() == [1, 0]
    es = t.model_from_descriptor({"model": "eight_schools"})
    assert es.dim == 10
    with pytest.raises(ValueError):
        t.model_from_descriptor({"model": "nope"})


def test_chunked_generator_matches_one_shot():
    """bench.py builds config 5 (8M x 255) with the chunked generator; it must
    reproduce tests_data.logistic_data exactly."""
    from tests_data import logistic_data, logistic_data_f32

    for n, p, chunk in ((10000, 255, 999), (4097, 54, 4096), (5, 3, 2)):
        x, y = logistic_data(n, p, 20191223)
        x32, y8 = logistic_data_f32(n, p, 20191223, chunk_rows=chunk)
        assert np.array_equal(x.astype(np.float32), x32)
        assert np.array_equal(y.astype(np.uint8), y8)
        for a, b in ((0, n // 3), (n // 3, n), (n // 2, n // 2 + 1)):
            xs, ys = logistic_data_f32(n, p, 20191223, chunk_rows=chunk, rows=(a, b))
            assert np.array_equal(xs, x32[a:b]) and np.array_equal(ys, y8[a:b])


def test_dense_gaussian_model_validation():
    with pytest.raises(ValueError):
        t.dense_gaussian_model(np.ones((3, 4)))
    with pytest.raises(ValueError):
        t.dense_gaussian_model(np.eye(3), inv_mass=-np.eye(3))
    with pytest.raises(ValueError):
        t.dense_gaussian_model(np.eye(3), precision="bf16")
    m = t.dense_gaussian_model(np.eye(4) * 2.0, inv_mass=np.eye(4) * 0.25, precision="fp64")
    assert m.name == "dense_gaussian" and m.dim == 4
    # x = L^-1 q with L = 0.5 I: A = L' P L = 0.5 I
    assert np.allclose(m.device_spec.params.reshape(4, 4), np.eye(4) * 0.5)
    assert np.allclose(m.device_spec.reparam, np.eye(4) * 0.5)


def test_oracle_dense_gaussian(oracle):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((40, 40))
    a = a @ a.T
    x = rng.standard_normal(40)
    m = oracle.Model("dense_gaussian", 40, dense_a=a.tolist())
    g = np.asarray(m.gradient(x.tolist()))
    assert np.allclose(g, a @ x, rtol=1e-12, atol=1e-12)
    assert np.isclose(m.potential(x.tolist()), 0.5 * x @ a @ x, rtol=1e-12)


def test_device_diagnostics_have_no_cpu_path():
    """chain_diagnostics_device runs the CUDA kernels only (no CPU fallback)."""
    import pytest
    import torch

    with pytest.raises((ValueError, RuntimeError)):
        t.ess_device(torch.zeros((2, 10, 3), dtype=torch.float64))


def test_pooled_covariance_has_no_cpu_path():
    import numpy as np
    import pytest

    import paper_1912_11554_b200 as t

    with pytest.raises((ValueError, RuntimeError)):
        t.pooled_covariance(np.zeros((4, 3)))


def test_logistic_data_keeps_fp64_when_not_fp32_exact():
    """No silent rounding (reference models.py:43-64 keeps fp64 X)."""
    x64 = np.array([[0.1, 1.0], [2.0, -3.0]])
    d = t.LogisticRegressionData(x64, [0, 1])
    assert d.x.dtype == np.float64 and not d.fp32_exact
    d32 = t.LogisticRegressionData(np.array([[0.5, 1.0], [2.0, -3.0]]), [0, 1])
    assert d32.x.dtype == np.float32 and d32.fp32_exact
