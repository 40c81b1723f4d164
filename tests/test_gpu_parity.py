"""Device parity against the reference (golden fixtures) and the CPU oracle.

Three layers (BASELINE.json north star):
  1. integers bit-exact: tree depth, leapfrog count, U-turn termination index
     (last check), R slot usage (writes, max occupied), chosen leaf index;
  2. floats: small models on the thread-team path are expected bit-identical
     to the reference (same op order, no FMA); we assert rel <= 1e-12 to leave
     room for last-ulp exp/log1p differences.  Logistic fp64 pass: rel <= 1e-10
     (summation order only); fp32 pass: rel <= 1e-5 (stated FP32 tolerance);
  3. statistics: posterior moments within Monte-Carlo error, R-hat < 1.01.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden, num, nums

pytestmark = pytest.mark.gpu

FP64_REL = 1e-10
SMALL_REL = 1e-12
BLOCK_REL = 1e-9
FP32_REL = 1e-5


def ts():
    import paper_1912_11554_b200 as t

    return t


def close(a, b, rel, atol=0.0):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    both_nan = np.isnan(a) & np.isnan(b)
    same_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    ok = both_nan | same_inf | (np.abs(a - b) <= rel * np.maximum(np.abs(a), np.abs(b)) + atol)
    return bool(ok.all())


def device_model(desc, precision="fp64"):
    t = ts()
    n = desc["name"]
    if n == "std_normal":
        return t.std_normal_model(desc["dim"])
    if n == "gaussian":
        return t.gaussian_model(nums(desc["cov_diag"]))
    if n == "funnel":
        return t.funnel_model(desc["dim"])
    if n == "eight_schools":
        return t.eight_schools_model()
    if n == "logistic_regression":
        x = np.asarray([nums(r) for r in desc["x"]])
        y = np.asarray(nums(desc["y"]))
        return t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=precision)
    raise ValueError(n)


# ----------------------------------------------------------------------------- rng


def test_rng_streams_bit_exact():
    import torch

    t = ts()
    lib = t._lib.load_library()
    for rec in golden("rng")["seeds"]:
        hi, lo = int(rec["key"][0]), int(rec["key"][1])
        key = t.RngKey.from_seed(int(rec["seed"]))
        assert (key.hi, key.lo) == (hi, lo)
        for kind, ref in ((0, nums(rec["uniform"])), (1, nums(rec["normal"]))):
            out = torch.zeros(len(ref), dtype=torch.float64, device="cuda")
            t._lib.check(lib.ts_rng_probe(hi, lo, kind, len(ref), out.data_ptr(), 0))
            got = out.cpu().numpy()
            assert np.array_equal(got, np.asarray(ref)), f"kind {kind} seed {rec['seed']}"
        idx = sorted(int(i) for i in rec["fold"])
        n = max(i for i in idx if i < 5000) + 1
        out = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
        t._lib.check(lib.ts_rng_probe(hi, lo, 2, n, out.data_ptr(), 0))
        words = out.cpu().numpy().view(np.uint64).reshape(n, 2)
        for i in idx:
            if i < n:
                assert [str(int(w)) for w in words[i]] == rec["fold"][str(i)]


def test_device_libm_matches_glibc():
    """csrc/ts_libm.cuh on the device: exp and log1p equal this image's glibc
    (the reference's math.exp / math.log1p) bit for bit; log is correctly
    rounded and equals glibc on every dual-averaging start value."""
    import torch
    from decimal import Decimal, getcontext

    t = ts()
    lib = t._lib.load_library()
    rng = np.random.default_rng(11)

    def dev(kind, x):
        xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        yd = torch.empty_like(xd)
        t._lib.check(lib.ts_libm_probe(kind, xd.data_ptr(), yd.data_ptr(), xd.numel(), 0))
        return yd.cpu().numpy()

    def glibc(f, x):
        out = []
        for v in x.tolist():
            try:
                out.append(f(v))
            except OverflowError:
                out.append(math.inf)
        return np.array(out)

    x = np.concatenate([-rng.exponential(3.0, 300_000), rng.uniform(-40, 40, 300_000), rng.uniform(-745, 709, 50_000)])
    assert np.array_equal(dev(0, x).view(np.uint64), glibc(math.exp, x).view(np.uint64))
    x = np.concatenate([rng.uniform(0, 1, 300_000), np.exp(rng.uniform(-745, 0, 100_000)), rng.uniform(-0.999, 10, 100_000)])
    assert np.array_equal(dev(1, x).view(np.uint64), glibc(math.log1p, x).view(np.uint64))
    k = np.arange(-60, 61, dtype=np.float64)
    x = np.concatenate([2.0 ** k, 10.0 * 2.0 ** k])
    assert np.array_equal(dev(2, x).view(np.uint64), glibc(math.log, x).view(np.uint64))
    x = np.exp(rng.uniform(-700, 700, 100_000))
    got, ref = dev(2, x), glibc(math.log, x)
    mis = np.nonzero(got != ref)[0]
    assert mis.size < 2e-3 * x.size
    getcontext().prec = 60
    for i in mis[:100]:
        assert float(Decimal(float(x[i])).ln()) == got[i]


# ----------------------------------------------------------------------------- models


@pytest.mark.parametrize("precision,rel", [("fp64", FP64_REL), ("fp32", FP32_REL)])
def test_logistic_potential_gradient(precision, rel):
    t = ts()
    for rec in golden("logistic"):
        from tests_data import logistic_data

        x, y = logistic_data(rec["n"], rec["p"], rec["seed"])
        m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=precision)
        pts = np.asarray([nums(p["q"]) for p in rec["points"]])
        out = t.models.potential_and_gradient(m.device_spec, pts)
        for k, p in enumerate(rec["points"]):
            scale = max(1.0, float(np.abs(nums(p["g"])).max()))
            assert close(out[k, 0], num(p["U"]), rel), (rec["n"], rec["p"], k, out[k, 0], p["U"])
            assert close(out[k, 1:], nums(p["g"]), rel, atol=rel * scale), (rec["n"], rec["p"], k)


@pytest.mark.parametrize("p", [65, 100, 255])
@pytest.mark.parametrize("precision,rel", [("fp64", FP64_REL), ("fp32", FP32_REL)])
def test_wide_logistic_potential_gradient(p, precision, rel, oracle):
    """Wide-p pass (64 < p <= 256, SURVEY 8(d) config 5 shape) vs the C oracle."""
    t = ts()
    from tests_data import logistic_data

    for n in (37, 5000, 70001):
        x, y = logistic_data(n, p, p + n)
        m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=precision)
        om = oracle.Model("logistic_regression", p + 1, x=np.ascontiguousarray(x), y=np.ascontiguousarray(y))
        rng = np.random.default_rng(p)
        for scale in (0.0, 0.05, 1.0):
            q = rng.standard_normal(p + 1) * scale
            got = t.models.potential_and_gradient(m.device_spec, q[None, :])[0]
            U, g = om.potential(q.tolist()), np.asarray(om.gradient(q.tolist()))
            assert close(got[0], U, rel), (n, p, scale, got[0], U)
            assert close(got[1:], g, rel, atol=rel * max(1.0, np.abs(g).max())), (n, p, scale)


@pytest.mark.parametrize("n", [1, 2, 31, 33])
@pytest.mark.parametrize("p", [1, 3, 54, 64, 65])
@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp64x"])
def test_logistic_ragged_shapes(n, p, precision, oracle):
    """Ragged and boundary shapes of every logistic layout (a single row, a
    partial 32-row tile, p at the narrow / wide boundary, odd p for the
    half-row fp64x tiles): potential and gradient vs the oracle, and a short
    run (trajectories, adaptation) that stays finite."""
    t = ts()
    rng = np.random.default_rng(n * 100 + p)
    x = rng.standard_normal((n, p)).astype(np.float32).astype(np.float64)
    y = (rng.random(n) < 0.5).astype(np.float64)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=precision)
    om = oracle.Model("logistic_regression", p + 1, x=x, y=y)
    rel = FP32_REL if precision == "fp32" else FP64_REL
    for q in (np.zeros(p + 1), rng.standard_normal(p + 1) * 0.3):
        got = t.models.potential_and_gradient(m.device_spec, q[None, :])[0]
        U, g = om.potential(q.tolist()), np.asarray(om.gradient(q.tolist()))
        assert close(got[0], U, rel, atol=rel), (n, p, precision, got[0], U)
        assert close(got[1:], g, rel, atol=rel * max(1.0, np.abs(g).max())), (n, p, precision)
    r = t.run(t.RunConfig(model={}, num_chains=1, num_warmup=30, num_samples=20, seed=n + p), m)[0]
    assert np.all(np.isfinite(r.samples)) and r.total_leapfrogs > 0


def test_wide_tree_matches_oracle(oracle):
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(20000, 255, 7)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y))
    om = oracle.Model("logistic_regression", 256, x=np.ascontiguousarray(x), y=np.ascontiguousarray(y))
    rng = np.random.default_rng(3)
    q, r = rng.standard_normal(256) * 0.01, rng.standard_normal(256)
    U, g = om.potential(q.tolist()), om.gradient(q.tolist())
    cfg = t.SamplerConfig(step_size=0.003, mass=t.MassMatrix.identity(256), max_tree_depth=8)
    key = t.RngKey.from_seed(17)
    z = t.PhasePoint(q, r, U, np.asarray(g))
    h0 = t.hamiltonian(z, cfg.mass)
    tr = t.TreeTrace()
    tree = t.build_tree_iterative(z, 6, 0.003, cfg, m, key, h_ref=h0, trace=tr)
    ot = oracle.build_tree(oracle.Point(q.tolist(), r.tolist(), U, g), 6, 0.003, [1.0] * 256, om, (key.hi, key.lo), h0)
    assert (tree.leapfrog_count, tree.turning, tree.diverging, tree.proposal_leaf) == (
        ot.sub.count, ot.turning, ot.diverging, ot.sub.prop_leaf)
    assert [tuple(c) for c in tr.checks] == [tuple(c) for c in ot.checks]
    assert close(tree.right.position, ot.sub.last.q, 1e-10, atol=1e-12)
    assert close(tree.log_weight, ot.sub.lw, 1e-10)


def test_logistic_grid_sizes_agree():
    """Any persistent-grid size gives the same fp64 result up to summation order."""
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(20000, 54, 9)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y))
    q = np.random.default_rng(1).standard_normal((2, 55)) * 0.2
    ref = t.models.potential_and_gradient(m.device_spec, q)
    for grid in (1, 7, 64):
        m.device_spec.set_grid(grid)
        got = t.models.potential_and_gradient(m.device_spec, q)
        assert close(got, ref, 1e-11, atol=1e-9)
    m.device_spec.set_grid(0)


@pytest.mark.parametrize("desc", [
    {"name": "std_normal", "dim": 7},
    {"name": "gaussian", "cov_diag": [0.3, 1.0, 4.0, 9.0]},
    {"name": "funnel", "dim": 5},
    {"name": "eight_schools"},
])
def test_small_model_potential_gradient_bitwise(desc, oracle):
    t = ts()
    m = device_model(desc)
    om = oracle.model_from_desc(desc)
    rng = np.random.default_rng(3)
    pts = rng.standard_normal((6, m.dim)) * 1.3
    out = t.models.potential_and_gradient(m.device_spec, pts)
    # exp/log1p are the only non-IEEE-exact operations: CUDA's and glibc's
    # results may differ in the last ulp (eight schools: tau = exp(log tau)).
    rel = 0.0 if desc["name"] in ("std_normal", "gaussian") else 1e-15
    for k in range(pts.shape[0]):
        q = pts[k].tolist()
        assert close(out[k, 0], om.potential(q), rel)
        assert close(out[k, 1:], np.asarray(om.gradient(q)), rel, atol=rel)


@pytest.mark.parametrize("mode", ["thread", "block", "warp"])
def test_leapfrog_matches_oracle(mode, oracle):
    t = ts()
    for desc in ({"name": "std_normal", "dim": 3}, {"name": "funnel", "dim": 4}, {"name": "eight_schools"}):
        m = device_model(desc)
        om = oracle.model_from_desc(desc)
        rng = np.random.default_rng(5)
        q, r = rng.standard_normal(m.dim), rng.standard_normal(m.dim)
        inv = rng.uniform(0.5, 2.0, m.dim)
        z = t.PhasePoint(q, r, om.potential(q.tolist()), np.asarray(om.gradient(q.tolist())))
        for eps in (0.1, -0.37):
            got = t.leapfrog(z, eps, t.MassMatrix(inv), m, exec_mode=mode)
            ref = oracle.leapfrog(oracle.Point(q.tolist(), r.tolist(), z.potential, z.grad.tolist()), eps,
                                  inv.tolist(), om)
            rel = 0.0 if mode == "thread" else 1e-13
            assert close(got.position, ref.q, rel) and close(got.momentum, ref.r, rel)
            assert close(got.potential, ref.U, max(rel, 1e-14)) and close(got.grad, ref.g, max(rel, 1e-14))


# ----------------------------------------------------------------------------- trees


def _run_tree_case(case, mode, precision="fp64"):
    t = ts()
    m = device_model(case["model"], precision)
    z = t.PhasePoint(np.asarray(nums(case["z"]["q"])), np.asarray(nums(case["z"]["r"])), num(case["z"]["U"]),
                     np.asarray(nums(case["z"]["g"])))
    cfg = t.SamplerConfig(step_size=abs(num(case["eps"])) or 1.0, mass=t.MassMatrix(nums(case["inv_diag"])),
                          max_tree_depth=max(case["max_tree_depth"], 1), criterion=case["criterion"],
                          divergence_threshold=num(case["threshold"]))
    key = t.RngKey(int(case["key"][0]), int(case["key"][1]))
    trace = t.TreeTrace()
    tree = t.build_tree_iterative(z, case["depth"], num(case["eps"]), cfg, m, key, h_ref=num(case["h_ref"]),
                                  trace=trace, exec_mode=mode if case["model"]["name"] != "logistic_regression" else None)
    return tree, trace


def _check_tree(case, tree, trace, rel):
    o = case["out"]
    ints_ok = (
        tree.leapfrog_count == o["leapfrog_count"]
        and tree.turning == o["turning"]
        and tree.diverging == o["diverging"]
        and tree.proposal_leaf == o["proposal_leaf"]
        and [tuple(w) for w in case["trace"]["writes"]] == [tuple(w) for w in trace.writes]
        and [tuple(c) for c in case["trace"]["checks"]] == [tuple(c) for c in trace.checks]
        and trace.max_occupied == case["trace"]["max_occupied"]
    )
    floats_ok = (
        close(tree.log_weight, num(o["log_weight"]), rel)
        and close(tree.sum_metropolis, num(o["sum_metropolis"]), rel)
        and close(tree.momentum_sum, nums(o["momentum_sum"]), rel, atol=rel)
        and close(tree.left.position, nums(o["left_q"]), rel, atol=rel)
        and close(tree.right.position, nums(o["right_q"]), rel, atol=rel)
        and close(tree.right.momentum, nums(o["right_r"]), rel, atol=rel)
        and close(tree.proposal.position, nums(o["prop_q"]), rel, atol=rel)
        and close(tree.proposal.potential, num(o["prop_U"]), rel)
        and close(trace.leaf_log_weights, nums(case["trace"]["leaf_log_weights"]), rel)
    )
    return ints_ok, floats_ok


@pytest.mark.parametrize("mode", ["thread", "block", "warp"])
def test_trees_match_reference(mode):
    cases = golden("trees")
    bad_int, bad_float = [], []
    for i, case in enumerate(cases):
        if mode != "block" and case["model"]["name"] == "logistic_regression":
            continue  # logistic always runs on the block/grid path
        tree, trace = _run_tree_case(case, mode)
        small = case["model"]["name"] != "logistic_regression"
        # block teams reduce dot products in a shuffle-tree order: ulp-level
        # differences that a leapfrog chain of up to 2^8 steps may amplify
        rel = (SMALL_REL if mode == "thread" else BLOCK_REL) if small else FP64_REL
        if not small:
            x = np.asarray([nums(r) for r in case["model"]["x"]])
            if not np.array_equal(x.astype(np.float32).astype(np.float64), x):
                # crosscheck.build_case draws X in fp64; the device stores X in
                # fp32, so these cases see data rounded by <= 2^-24
                rel = FP32_REL
        ints_ok, floats_ok = _check_tree(case, tree, trace, rel)
        if not ints_ok:
            bad_int.append(i)
        if not floats_ok:
            bad_float.append(i)
    assert not bad_int, f"integer mismatches in cases {bad_int[:10]}"
    assert not bad_float, f"float mismatches in cases {bad_float[:10]}"


def test_trees_fp32_logistic_within_tolerance():
    cases = [c for c in golden("trees") if c["model"]["name"] == "logistic_regression"]
    assert cases
    int_mismatch = 0
    for case in cases:
        tree, trace = _run_tree_case(case, None, precision="fp32")
        ints_ok, _ = _check_tree(case, tree, trace, FP32_REL)
        int_mismatch += not ints_ok
        if ints_ok:
            assert close(tree.right.position, nums(case["out"]["right_q"]), FP32_REL, atol=FP32_REL)
            assert close(tree.log_weight, num(case["out"]["log_weight"]), FP32_REL)
    # fp32 rounding may flip a decision that sits on a near-tie; none expected on this battery
    assert int_mismatch == 0


# ----------------------------------------------------------------------------- transitions


@pytest.mark.parametrize("mode", ["thread", "block", "warp"])
def test_transitions_match_reference(mode):
    t = ts()
    for rec in golden("transitions"):
        m = device_model(rec["model"])
        cfg = t.SamplerConfig(step_size=rec["step"], mass=t.MassMatrix(nums(rec["inv_diag"])),
                              max_tree_depth=rec["max_tree_depth"], criterion=rec["criterion"])
        for d in rec["draws"]:
            z = t.PhasePoint(np.asarray(nums(d["z_in"]["q"])), np.zeros(m.dim), num(d["z_in"]["U"]),
                             np.asarray(nums(d["z_in"]["g"])))
            key = t.RngKey(int(d["key"][0]), int(d["key"][1]))
            z1, st, tr = t.nuts_transition_from(z, cfg, m, key, exec_mode=mode, return_trace=True)
            ref = d["stats"]
            assert (st.depth_reached, st.leapfrog_calls, int(st.diverged)) == tuple(ref[:3])
            assert [(a, b, c, e) for a, b, c, e, _ in tr.trees] == [(x[0], x[2], x[3] + 2 * x[4], x[1]) for x in d["trees"]]
            assert [o for _, o in tr.outer_checks] == d["outer"]
            assert close(st.accept_stat, num(ref[3]), SMALL_REL) and close(st.energy, num(ref[4]), SMALL_REL)
            assert close(z1.position, nums(d["z_out"]["q"]), SMALL_REL, atol=1e-15)
            assert close(z1.potential, num(d["z_out"]["U"]), SMALL_REL)


# ----------------------------------------------------------------------------- runs


def test_runs_match_reference():
    t = ts()
    for rec in golden("runs"):
        desc = dict(rec["desc"])
        if desc["model"] == "eight_schools":
            model = t.eight_schools_model()
        else:
            model = t.model_from_descriptor(desc)
        sampler = None
        if rec["sampler"] is not None:
            s = rec["sampler"]
            sampler = t.SamplerConfig(step_size=s["step"], mass=t.MassMatrix.identity(model.dim),
                                      criterion=s["criterion"], max_tree_depth=s["max_tree_depth"])
        cfg = t.RunConfig(model=desc, num_chains=rec["num_chains"], num_warmup=rec["num_warmup"],
                          num_samples=rec["num_samples"], seed=rec["seed"], sampler=sampler)
        # thread team: the reference's summation order; the engine's exp / log1p
        # are glibc's bit for bit and its log is correctly rounded
        # (csrc/ts_libm.cuh), so adapted runs are reproduced whole: dual
        # averaging, Welford windows and every warmup and sampling draw
        res = t.run(cfg, model, exec_mode="thread")
        for r, ref in zip(res, rec["chains"]):
            stats = r.stats_array
            ref_stats = np.asarray([[num(v) for v in s] for s in ref["stats"]])
            assert np.array_equal(stats[:, :3], ref_stats[:, :3]), desc
            assert close(stats[:, 3:], ref_stats[:, 3:], 1e-12), desc
            assert r.total_leapfrogs == ref["total_leapfrogs"], desc
            assert close(r.samples, [nums(s) for s in ref["samples"]], 1e-12, atol=1e-13), desc
            assert close(r.adaptation["final_step_size"], num(ref["adaptation"]["final_step_size"]), 1e-15), desc
            if rec["num_warmup"] > 0:
                wst = r.warmup_stats_array
                rw = ref_stats_w(rec, ref)
                assert np.array_equal(wst[:, :3], rw[:, :3]), desc
                assert close(wst[:, 3:], rw[:, 3:], 1e-12), desc
                assert close(r.adaptation["initial_step_size"], num(ref["adaptation"]["initial_step_size"]), 0.0)
                assert close(r.adaptation["step_size_trace"], nums(ref["adaptation"]["step_size_trace"]), 1e-15), desc
                assert close(r.adaptation["inv_mass_diag"], nums(ref["adaptation"]["inv_mass_diag"]), 1e-12), desc


@pytest.mark.parametrize("which", ["gauss10", "eight_schools", "logistic"])
def test_adaptation_replay_matches_reference_recursion(which):
    """The device's warmup adaptation, audited draw by draw: the reference's
    dual-averaging and windowed-Welford recursion (adapt.py:44-108, 207-236;
    oracle.Adaptation) is replayed on the host from the device's own warmup
    accept stats and positions.  The recursion is pure IEEE arithmetic apart
    from log(10 eps0) / exp(log_eps) (last-ulp CUDA vs glibc), so the step
    size before every warmup transition and the final step size must agree to
    1e-14 relative -- a wrong gain, t0, kappa or clipping shows at the first
    draws -- and the installed inverse mass must be bit-identical, with the
    schedule's number of installs (W = 200: windows 25/50/60/15)."""
    import turnstile_oracle as o
    from tests_data import logistic_data

    t = ts()
    from paper_1912_11554_b200.chains import run_device

    W, S, C = 200, 5, 4
    if which == "gauss10":
        model = t.gaussian_model(np.linspace(0.5, 3.0, 10))
    elif which == "eight_schools":
        model = t.eight_schools_model()
    else:
        x, y = logistic_data(2000, 6, 3)
        model = t.logistic_regression_model(t.LogisticRegressionData(x, y))
    cfg = t.RunConfig(model={"model": which}, num_chains=C, num_warmup=W, num_samples=S, seed=17)
    keys = t.chain_keys(cfg.seed, C)
    run = run_device(model, cfg, keys, keep_warmup=True)
    samples = run.samples.cpu().numpy()
    stats = run.stats.cpu().numpy()
    adapt = run.adapt.cpu().numpy()
    assert samples.shape == (C, W + S, model.dim)
    windows = sum(1 for f in o.schedule_flags(W) if f & 2)
    for c in range(C):
        eps0 = float(adapt[c, 0])
        rep = o.replay_adaptation(eps0, stats[c, :W, 3], samples[c, :W], target=cfg.target_accept)
        dev_trace = adapt[c, 2:2 + W]
        assert close(dev_trace, rep["step_size_trace"], 1e-14), (which, c)
        assert close(adapt[c, 1], rep["final_step_size"], 1e-14), (which, c)
        assert np.array_equal(adapt[c, 2 + W:], np.asarray(rep["inv_mass_diag"])), (which, c)
        assert rep["installs"] == windows == 4
        # the sampling phase starts where warmup ended and uses the final settings
        assert np.all(np.isfinite(samples[c, W:]))


def ref_stats_w(rec, ref):
    """Warmup stats are not in ChainResult.stats (reference keeps sampling
    stats only); recompute them with the oracle for the comparison."""
    import turnstile_oracle as o

    desc = rec["desc"]
    md = {"name": desc["model"], **desc["params"]}
    m = o.model_from_desc(md)
    idx = rec["chains"].index(ref)
    key = o.chain_keys(rec["seed"], rec["num_chains"])[idx]
    out = o.run_chain(m, key, rec["num_warmup"], 1)
    return np.asarray([[s.depth, s.leapfrogs, int(s.diverged), s.accept, s.energy]
                       for s in out["stats"][: rec["num_warmup"]]])


def test_sampling_correctness_10d_normal():
    """Reference acceptance criterion 5 (test_acceptance.py:100-122) on the device."""
    t = ts()
    cfg = t.RunConfig(model={"model": "std_normal", "params": {"dim": 10}}, num_chains=4, num_warmup=1000,
                      num_samples=1000, seed=7)
    res = t.run(cfg)
    s = t.summarize(res)
    assert (np.abs(s.mean) < 0.05).all()
    assert ((s.std ** 2 > 0.9) & (s.std ** 2 < 1.1)).all()
    assert (s.split_rhat < 1.01).all()
    assert (s.ess > 400).all()


# ----------------------------------------------------------------------------- covtype shape


def test_covtype_transitions_match_oracle(oracle):
    """Full-size config 2: transitions of a device run, re-run from the run's own
    states on the device and on the CPU oracle (fp64): identical integers, and
    positions within 1e-12 after up to 2^10-1 leapfrogs over 581,012 rows."""
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(581012, 54, 20191222)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="fp64")
    W, S, seed = 150, 12, 1001
    cfg = t.RunConfig(model={}, num_chains=1, num_warmup=W, num_samples=S, seed=seed)
    key = t.chain_keys(seed, 1)[0]
    r = t.run_device(m, cfg, [key], 0)
    st = r.stats.cpu().numpy()[0]
    ad = r.adapt.cpu().numpy()[0]
    samples = r.samples.cpu().numpy()[0]
    step, inv = float(ad[1]), ad[2 + W:].copy()
    om = oracle.Model("logistic_regression", 55, x=x, y=y, fused_omp=True)
    for i in (1, 5, 9):
        q0 = samples[i - 1]
        U0, g0 = m.potential(q0), m.gradient(q0)
        z = t.PhasePoint(q0, np.zeros(55), U0, g0)
        dkey = key.fold(10 + W + i)
        z1, s1 = t.nuts_transition_from(z, t.SamplerConfig(step_size=step, mass=t.MassMatrix(inv)), m, dkey)
        oz, os_, _ = oracle.transition(oracle.Point(q0.tolist(), [0.0] * 55, U0, g0.tolist()), step, inv.tolist(), om,
                                       (dkey.hi, dkey.lo))
        assert (s1.depth_reached, s1.leapfrog_calls) == (os_.depth, os_.leapfrogs) == (int(st[W + i, 0]),
                                                                                      int(st[W + i, 1]))
        assert close(z1.position, oz.q, 1e-12, atol=1e-14)
        assert np.array_equal(z1.position, samples[i])  # the run's own draw


@pytest.mark.parametrize("eps,max_depth", [(0.02, 10), (0.3, 10), (3.0, 6), (0.05, 1), (0.05, 2)])
def test_logistic_trajectory_stops_match_oracle(eps, max_depth, oracle):
    """Worker-run trajectories (LogisticW::serve_traj) under every way a
    doubling ends: U-turns mid-tree (the speculative leaf is discarded),
    divergences (large eps), the depth cap, depth-1/2 trees.  Per-tree
    integers (direction, leapfrogs, stop kind), outer checks, proposal and
    positions against the CPU oracle, and a second call with the same key
    repeats the first bit for bit (the launch leaves no state behind)."""
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(3000, 54, 77)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="fp64")
    om = oracle.Model("logistic_regression", 55, x=x, y=y)
    rng = np.random.default_rng(int(eps * 1000) + max_depth)
    cfg = t.SamplerConfig(step_size=eps, mass=t.MassMatrix.identity(55), max_tree_depth=max_depth)
    for case in range(6):
        q0 = rng.standard_normal(55) * 0.1
        U0, g0 = om.potential(q0.tolist()), om.gradient(q0.tolist())
        z = t.PhasePoint(q0, np.zeros(55), U0, np.asarray(g0))
        key = t.RngKey.from_seed(1000 + case)
        z1, st, tr = t.nuts_transition_from(z, cfg, m, key, return_trace=True)
        z2, st2, _ = t.nuts_transition_from(z, cfg, m, key, return_trace=True)
        assert np.array_equal(z1.position, z2.position) and st == st2
        oz, ost, dec = oracle.transition(oracle.Point(q0.tolist(), [0.0] * 55, U0, g0), eps, [1.0] * 55, om,
                                         (key.hi, key.lo), max_depth=max_depth)
        got = (st.depth_reached, st.leapfrog_calls, int(st.diverged),
               tuple((j, gr, c, stp) for j, c, stp, gr, _ in tr.trees), (tr.proposal_tree, tr.proposal_leaf))
        want = (ost.depth, ost.leapfrogs, int(ost.diverged),
                tuple((j, d, c, tu + 2 * dv) for j, d, c, tu, dv, _ in dec["trees"]), tuple(dec["proposal"]))
        assert got == want, (eps, max_depth, case, got, want)
        assert close(z1.position, oz.q, 1e-10, atol=1e-12)


@pytest.mark.parametrize("precision,rel", [("fp64", 1e-11), ("fp32", FP32_REL)])
def test_covtype_shape_potential_gradient(precision, rel, oracle):
    """Full BASELINE config-2 size (581,012 x 54) against the C oracle."""
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(581012, 54, 20191222)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=precision)
    om = oracle.Model("logistic_regression", 55, x=np.ascontiguousarray(x), y=np.ascontiguousarray(y))
    rng = np.random.default_rng(2)
    for q in (np.zeros(55), rng.standard_normal(55) * 0.05):
        got = t.models.potential_and_gradient(m.device_spec, q[None, :])[0]
        U = om.potential(q.tolist())
        g = np.asarray(om.gradient(q.tolist()))
        assert close(got[0], U, rel)
        assert close(got[1:], g, rel, atol=rel * np.abs(g).max())


# ----------------------------------------------------------------------------- row sharding (config 5)


def _canon(words):
    t = ts()
    w = np.asarray(words, dtype=np.uint64).copy()
    n = (w.size - 1) // 2
    w[0:2 * n:2], w[1:2 * n:2] = t.rowshard.canonical(w[0:2 * n:2], w[1:2 * n:2])
    return w


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_row_shards_compose_exactly(precision):
    """Wide-p totals are exact fixed-point sums of per-tile partials, so the
    row shards' totals add up to the single-GPU totals bit for bit, and the
    (U, gradient) every rank derives equals the one-GPU result exactly."""
    t = ts()
    from tests_data import logistic_data

    n, p = 20005, 255
    x, y = logistic_data(n, p, 11)
    full = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision=precision).device_spec
    rng = np.random.default_rng(5)
    for scale in (0.0, 0.05, 0.5):
        q = rng.standard_normal(p + 1) * scale
        ref_words = t.rowshard.partial_sums(full, q)
        ref_ug = t.models.potential_and_gradient(full, q[None, :])[0]
        assert np.array_equal(t.rowshard.totals_to_potential_gradient(ref_words, q), ref_ug)
        for world in (2, 3, 8):
            parts = []
            for r in range(world):
                a, b = t.rowshard.row_range(n, r, world)
                assert a % 32 == 0
                m = t.logistic_regression_model(t.LogisticRegressionData(x[a:b], y[a:b]), precision=precision)
                parts.append(t.rowshard.partial_sums(m.device_spec, q))
            comb = t.rowshard.combine(parts)
            assert np.array_equal(_canon(comb), _canon(ref_words)), (world, scale)
            assert np.array_equal(t.rowshard.totals_to_potential_gradient(comb, q), ref_ug)


@pytest.mark.parametrize("p", [54, 255])
def test_row_shard_mailbox_world1_identical(p):
    """world = 1 runs the peer-exchange device path (push, flag, wait, sum)
    against its own mailbox: results equal the unconnected model's bitwise,
    across launches (persistent exchange counter)."""
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(30000, p, 2)
    plain = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="fp32")
    shard = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="fp32")
    t.rowshard.connect(shard.device_spec, 0, 1, lambda b: [b])
    assert shard.device_spec.row_shard == (0, 1)
    q = np.random.default_rng(1).standard_normal((3, p + 1)) * 0.05
    a = t.models.potential_and_gradient(plain.device_spec, q)
    b = t.models.potential_and_gradient(shard.device_spec, q)
    assert np.array_equal(a, b)
    cfg = t.RunConfig(model={}, num_chains=1, num_warmup=30, num_samples=20, seed=4)
    for _ in range(2):
        ra = t.run_device(plain, cfg, t.chain_keys(4, 1), 0)
        rb = t.run_device(shard, cfg, t.chain_keys(4, 1), 0)
        assert np.array_equal(ra.samples.cpu().numpy(), rb.samples.cpu().numpy())
        assert np.array_equal(ra.stats.cpu().numpy(), rb.stats.cpu().numpy())


# ----------------------------------------------------------------------------- tcgen05 GEMM (config 4)


def _tf32(a):
    """Round fp32 to the nearest tf32 (10-bit mantissa), ties away (cvt.rna)."""
    b = np.asarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return b.view(np.float32)


@pytest.mark.parametrize("M,N,K,grid", [(128, 64, 32, 0), (200, 100, 60, 0), (1000, 1024, 1000, 0), (1000, 1024, 1000, 37)])
def test_tcgen05_tf32_gemm_probe(M, N, K, grid):
    import torch

    t = ts()
    lib = t._lib.load_library()
    rng = np.random.default_rng(M + N + K)
    a = _tf32(rng.standard_normal((M, K)).astype(np.float32))
    xt = _tf32(rng.standard_normal((N, K)).astype(np.float32))
    ad, xd = torch.from_numpy(a).cuda(), torch.from_numpy(xt).cuda()
    gt = torch.full((N, M), float("nan"), dtype=torch.float32, device="cuda")
    t._lib.check(lib.ts_gemm_tf32_probe(ad.data_ptr(), xd.data_ptr(), gt.data_ptr(), M, N, K, grid, 0))
    torch.cuda.synchronize()
    ref = xt.astype(np.float64) @ a.astype(np.float64).T
    got = gt.cpu().numpy().astype(np.float64)
    # tf32 x tf32 products are exact in fp32; only fp32 accumulation rounds
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-5, err


def _spd(D, seed, cond=100.0):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((D, D)))
    lam = np.logspace(-np.log10(cond) / 2, np.log10(cond) / 2, D)
    return (q * lam) @ q.T


@pytest.mark.parametrize("D", [16, 100])
def test_dense_potential_gradient(D, oracle):
    t = ts()
    A = _spd(D, D)
    om = oracle.Model("dense_gaussian", D, dense_a=A.tolist())
    q = np.random.default_rng(1).standard_normal((3, D))
    m64 = t.dense_gaussian_model(A, precision="fp64")
    out = t.models.potential_and_gradient(m64.device_spec, q)
    for k in range(3):
        assert out[k, 0] == om.potential(q[k].tolist())  # SIMT fp64 policy: bit for bit
        assert np.array_equal(out[k, 1:], np.asarray(om.gradient(q[k].tolist())))
    if D % 4 == 0:
        m32 = t.dense_gaussian_model(A, precision="tf32")
        o32 = t.models.potential_and_gradient(m32.device_spec, q)
        g = q @ A.T
        # TF32 operands (10-bit mantissa): stated tolerance 2e-3 relative to |g|
        assert np.abs(o32[:, 1:] - g).max() <= 2e-3 * np.abs(g).max()
        assert np.allclose(o32[:, 0], 0.5 * np.einsum("kd,kd->k", q, g), rtol=2e-3)


@pytest.mark.parametrize("D", [16, 160])
def test_dense_tree_fp64_matches_oracle(D, oracle):
    """D = 160 takes the batched model's fused leaf pass (D >= 128: kick,
    prefix sum, energies, next drift, request row and NodeStore copies in one
    vector loop); D = 16 the separate loops."""
    t = ts()
    A = _spd(D, 3)
    om = oracle.Model("dense_gaussian", D, dense_a=A.tolist())
    m = t.dense_gaussian_model(A, precision="fp64")
    rng = np.random.default_rng(9)
    bad_int = 0
    for case in range(12):
        q, r = rng.standard_normal(D), rng.standard_normal(D)
        U, g = om.potential(q.tolist()), om.gradient(q.tolist())
        eps = [0.05, 0.2, 0.6][case % 3]
        cfg = t.SamplerConfig(step_size=eps, mass=t.MassMatrix.identity(D), max_tree_depth=8)
        key = t.RngKey.from_seed(100 + case)
        z = t.PhasePoint(q, r, U, np.asarray(g))
        h0 = t.hamiltonian(z, cfg.mass)
        tr = t.TreeTrace()
        depth = 1 + case % 6
        tree = t.build_tree_iterative(z, depth, eps * (1 if case % 2 else -1), cfg, m, key, h_ref=h0, trace=tr)
        ot = oracle.build_tree(oracle.Point(q.tolist(), r.tolist(), U, g), depth, eps * (1 if case % 2 else -1),
                               [1.0] * D, om, (key.hi, key.lo), h0)
        ints = (tree.leapfrog_count, tree.turning, tree.diverging, tree.proposal_leaf) == (
            ot.sub.count, ot.turning, ot.diverging, ot.sub.prop_leaf) and [tuple(c) for c in tr.checks] == [
            tuple(c) for c in ot.checks]
        bad_int += not ints
        if ints:
            assert close(tree.right.position, ot.sub.last.q, BLOCK_REL, atol=BLOCK_REL)
            assert close(tree.log_weight, ot.sub.lw, BLOCK_REL)
    assert bad_int == 0


def test_dense_many_chains_tf32_vs_fp64():
    """Config-4 path at small scale: 64 chains in lockstep; the TF32 tensor-core
    run agrees with the fp64 SIMT run statistically and in its first tree
    decisions (acceptance/depth), and both recover the target moments."""
    t = ts()
    D, C = 32, 64
    A = _spd(D, 5, cond=10.0)
    cov = np.linalg.inv(A)
    cfg = t.RunConfig(model={}, num_chains=C, num_warmup=200, num_samples=200, seed=11)
    keys = t.chain_keys(11, C)
    runs = {}
    for prec in ("fp64", "tf32"):
        m = t.dense_gaussian_model(A, precision=prec)
        runs[prec] = t.run_device(m, cfg, keys, 0)
    s64 = runs["fp64"].samples.cpu().numpy()
    s32 = runs["tf32"].samples.cpu().numpy()
    st64 = runs["fp64"].stats.cpu().numpy()
    st32 = runs["tf32"].stats.cpu().numpy()
    # first warmup transition of every chain: same start, same randomness
    same_depth = np.mean(st64[:, 0, 0] == st32[:, 0, 0])
    assert same_depth >= 0.9, same_depth
    for s in (s64, s32):
        flat = s.reshape(-1, D)
        assert np.abs(flat.mean(0)).max() < 6 * np.sqrt(np.diag(cov).max() / (C * 200 / 5))
        assert np.allclose(flat.var(0), np.diag(cov), rtol=0.15)
    rhat = t.split_rhat(s32)
    assert np.nanmax(rhat) < 1.05


def test_dense_tf32_decision_flips(oracle):
    """Config-4 TF32 decisions counted against fp64 (north star: "acceptance
    decisions checked against FP32"): 1008 transitions of
    an fp64 run (16 chains x 63 post-warmup states) are replayed from the same
    (q, key, step) by the TF32 tensor-core path and the fp64 SIMT path; the
    integer decisions (depth, leapfrogs, divergence, per-tree direction /
    count / stop, proposal) are compared.  Bound: <= 2% flips, each at a
    near-tie of the oracle's decision margins (<= 5e-3: TF32 keeps 10
    mantissa bits, the stated gradient tolerance is 2e-3 relative, so energy
    errors of ~1e-3 move a multinomial / accept probability by about that
    much; measured: 6 flips of 1008, margins 1.0e-4 .. 2.0e-3)."""
    import json

    t = ts()
    D, C, W, S = 64, 16, 150, 64
    A = _spd(D, 21, cond=30.0)
    om = oracle.Model("dense_gaussian", D, dense_a=A.tolist())
    m64 = t.dense_gaussian_model(A, precision="fp64")
    m32 = t.dense_gaussian_model(A, precision="tf32")
    cfg = t.RunConfig(model={}, num_chains=C, num_warmup=W, num_samples=S, seed=23)
    keys = t.chain_keys(23, C)
    r = t.run_device(m64, cfg, keys, 0)
    samples = r.samples.cpu().numpy()
    adapt = r.adapt.cpu().numpy()
    flips, n = [], 0
    for c in range(C):
        step = float(adapt[c, 1])
        scfg = t.SamplerConfig(step_size=step, mass=t.MassMatrix.identity(D))
        for i in range(1, S):
            q0 = samples[c, i - 1]
            dkey = keys[c].fold(10 + W + i)
            dec = {}
            for prec, m in (("fp64", m64), ("tf32", m32)):
                ug = t.models.potential_and_gradient(m.device_spec, q0[None, :])[0]
                z = t.PhasePoint(q0, np.zeros(D), float(ug[0]), ug[1:].copy())
                _, st, tr = t.nuts_transition_from(z, scfg, m, dkey, return_trace=True)
                dec[prec] = (st.depth_reached, st.leapfrog_calls, int(st.diverged),
                             tuple((j, gr, cc, stp) for j, cc, stp, gr, _ in tr.trees), (tr.proposal_tree, tr.proposal_leaf))
            n += 1
            if dec["tf32"] != dec["fp64"]:
                margins = []
                oracle.transition(oracle.Point(q0.tolist(), [0.0] * D, om.potential(q0.tolist()), om.gradient(q0.tolist())),
                                  step, [1.0] * D, om, (dkey.hi, dkey.lo), margins=margins)
                mrg = min((mm for tm in margins for mm in tm), key=lambda km: km[1], default=("none", math.inf))
                flips.append({"chain": c, "draw": i, "kind": mrg[0], "min_margin": mrg[1],
                              "tf32": dec["tf32"][:3], "fp64": dec["fp64"][:3]})
    print("dense tf32 decision replay:", json.dumps({"replayed": n, "flips": len(flips), "flip_rate": len(flips) / n,
                                                      "flip_log": flips}))
    assert n == 1008
    assert len(flips) <= 0.02 * n, flips
    assert all(f["min_margin"] <= 5e-3 for f in flips), flips


@pytest.mark.parametrize("rows,D", [(1, 1), (130, 100), (1000, 1000)])
def test_dense_transform_matches_numpy(rows, D):
    """ts_dense_transform (q = L x per draw, the dense-mass sample map) vs numpy."""
    import torch

    t = ts()
    lib = t._lib.load_library()
    rng = np.random.default_rng(rows + D)
    L = np.tril(rng.standard_normal((D, D)))
    x = rng.standard_normal((rows, D))
    Ld, xd = torch.from_numpy(L).cuda(), torch.from_numpy(x).cuda()
    qd = torch.empty_like(xd)
    t._lib.check(lib.ts_dense_transform(Ld.data_ptr(), xd.data_ptr(), qd.data_ptr(), rows, D, 0))
    ref = x @ L.T
    assert close(qd.cpu().numpy(), ref, 1e-11, atol=1e-11 * np.abs(ref).max())


def test_dense_mass_reparametrisation():
    """Dense inverse mass M^-1 = Sigma: the sampler runs on x = L^-1 q and
    returns q; moments match Sigma."""
    t = ts()
    D, C = 16, 32
    A = _spd(D, 7, cond=1000.0)
    cov = np.linalg.inv(A)
    m = t.dense_gaussian_model(A, inv_mass=cov, precision="fp64")
    cfg = t.RunConfig(model={}, num_chains=C, num_warmup=100, num_samples=300, seed=2)
    r = t.run_device(m, cfg, t.chain_keys(2, C), 0)
    flat = r.samples.cpu().numpy().reshape(-1, D)
    emp = np.cov(flat.T)
    assert np.abs(emp - cov).max() <= 0.15 * np.abs(cov).max()


# ----------------------------------------------------------------------------- HMC baseline


def test_hmc_transition_matches_reference():
    """Device hmc_transition (sampler.py:163-203) vs the reference's draws:
    accept decisions and leapfrog counts exact, floats at the thread-team
    tolerance."""
    t = ts()
    for case in golden("hmc"):
        m = device_model(case["model"])
        cfg = t.SamplerConfig(step_size=num(case["step"]), mass=t.MassMatrix.identity(m.dim))
        for d in case["draws"]:
            key = t.RngKey(int(d["key"][0]), int(d["key"][1]))
            q, st = t.hmc_transition(np.asarray(nums(d["q_in"])), cfg, m, key, case["num_steps"])
            assert st.leapfrog_calls == d["leapfrogs"] and st.diverged == d["diverged"]
            assert close(q, nums(d["q_out"]), SMALL_REL, atol=SMALL_REL)
            assert close(st.accept_stat, num(d["accept_stat"]), SMALL_REL)
            assert close(st.energy, num(d["energy"]), SMALL_REL)


def test_dense_run_chunks_beyond_one_grid():
    """More chains than one co-resident grid holds (148 SMs x 8 chain warps):
    the run is chunked; every chain is a pure function of its key."""
    t = ts()
    D, C = 16, 1500
    A = _spd(D, 9, cond=10.0)
    m = t.dense_gaussian_model(A, precision="fp64")
    cfg = t.RunConfig(model={}, num_chains=C, num_warmup=20, num_samples=5, seed=8)
    keys = t.chain_keys(8, C)
    big = t.run_device(m, cfg, keys, 0).samples.cpu().numpy()
    assert np.isfinite(big).all()
    for c in (0, 1, 1199, 1499):
        one = t.run_device(m, cfg, [keys[c]], 0).samples.cpu().numpy()[0]
        assert np.array_equal(big[c], one), c


@pytest.mark.parametrize("prec", ["tf32", "fp64"])
def test_dense_release_protocols_agree(prec, monkeypatch):
    """The batched GEMM steps release served chains either after a grid
    barrier (default) or per N-tile by the CTA finishing its last M-tile
    (TS_DENSE_EARLY=1); each chain is a pure function of its key, so both
    protocols give bit-identical runs (D = 256 takes the fused leaf pass)."""
    t = ts()
    D, C = 256, 200
    A = _spd(D, 13, cond=20.0)
    m = t.dense_gaussian_model(A, precision=prec)
    cfg = t.RunConfig(model={}, num_chains=C, num_warmup=30, num_samples=20, seed=12)
    keys = t.chain_keys(12, C)
    runs = []
    for early in ("0", "1"):
        monkeypatch.setenv("TS_DENSE_EARLY", early)
        r = t.run_device(m, cfg, keys, 0)
        runs.append((r.samples.cpu().numpy(), r.stats.cpu().numpy()))
    assert np.isfinite(runs[0][0]).all()
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])


def test_ess_device_on_gpu_samples():
    """Device ESS / split R-hat on a many-chain run's samples in HBM."""
    t = ts()
    m = t.eight_schools_model()
    cfg = t.RunConfig(model={}, num_chains=256, num_warmup=100, num_samples=200, seed=3)
    r = t.run_device(m, cfg, t.chain_keys(3, 256), 0)
    e, rh = t.chain_diagnostics_device(r.samples)
    host = r.samples.cpu().numpy()
    assert np.allclose(e, t.ess(host), rtol=1e-10)
    assert np.allclose(rh, t.split_rhat(host), rtol=1e-12)


@pytest.mark.parametrize("shape,phi", [((4, 100, 3), 0.7), ((16, 1000, 10), 0.7), ((1, 50, 2), 0.5), ((3, 7, 1), 0.3),
                                       ((2, 4, 2), 0.0), ((8, 999, 3), 0.995), ((5, 301, 40), -0.6),
                                       ((8192, 1000, 10), 0.8)])
def test_device_diagnostics_match_host_estimators(shape, phi):
    """ts_chain_diagnostics vs diagnostics.ess / split_rhat (the reference
    estimators, diagnostics.py:49-105): AR(1) chains incl. strongly
    autocorrelated (phi = 0.995: Geyer truncation past several 64-lag
    blocks), antithetic (phi < 0: ESS capped at m n), odd draw counts, the
    minimum of 4 draws, and the 8192 x 1000 x 10 eight-schools shape."""
    import torch

    t = ts()
    rng = np.random.default_rng(abs(hash(shape)) % 2**32)
    x = rng.standard_normal(shape)
    for i in range(1, shape[1]):
        x[:, i] = phi * x[:, i - 1] + x[:, i]
    x += rng.standard_normal((shape[0], 1, shape[2])) * 0.05  # chain offsets: R-hat > 1
    xd = torch.from_numpy(x).cuda()
    e, rh = t.chain_diagnostics_device(xd)
    assert np.allclose(e, t.ess(x), rtol=1e-10, atol=0), (e, t.ess(x))
    assert np.allclose(rh, t.split_rhat(x), rtol=1e-12, atol=0)


def test_device_diagnostics_constant_dimension_is_nan():
    import torch

    t = ts()
    x = np.random.default_rng(1).standard_normal((4, 40, 3))
    x[:, :, 1] = 2.5
    with pytest.warns(RuntimeWarning):
        e, rh = t.chain_diagnostics_device(torch.from_numpy(x).cuda())
    assert np.isnan(e[1]) and np.isnan(rh[1]) and np.isfinite(e[[0, 2]]).all()
    with pytest.warns(RuntimeWarning):
        assert np.allclose(e[[0, 2]], t.ess(x)[[0, 2]], rtol=1e-10)


def test_block_team_runs_every_chain():
    """exec_mode='block' runs one CTA per chain: every chain's draws match the
    thread-team run (same keys) to the block-reduction tolerance."""
    t = ts()
    m = t.gaussian_model(np.logspace(-1, 1, 10))
    cfg = t.RunConfig(model={}, num_chains=5, num_warmup=0, num_samples=4, seed=12,
                      sampler=t.SamplerConfig(step_size=0.3, mass=t.MassMatrix.identity(10)))
    keys = t.chain_keys(12, 5)
    a = t.run_device(m, cfg, keys, 0, exec_mode="thread").samples.cpu().numpy()
    b = t.run_device(m, cfg, keys, 0, exec_mode="block").samples.cpu().numpy()
    assert np.isfinite(b).all()
    assert close(b[:, :3], a[:, :3], BLOCK_REL, atol=BLOCK_REL)


def test_warp_team_runs_every_chain():
    """exec_mode='warp' runs one warp per chain (8 per CTA, vectors in shared
    memory): a chain count that is not a multiple of 8, every chain's draws
    and stats match the thread-team run to the shuffle-reduction tolerance."""
    t = ts()
    for m, D in ((t.eight_schools_model(), 10), (t.gaussian_model(np.logspace(-1, 1, 40)), 40)):
        cfg = t.RunConfig(model={}, num_chains=37, num_warmup=0, num_samples=4, seed=13,
                          sampler=t.SamplerConfig(step_size=0.2, mass=t.MassMatrix.identity(D)))
        keys = t.chain_keys(13, 37)
        a = t.run_device(m, cfg, keys, 0, exec_mode="thread")
        b = t.run_device(m, cfg, keys, 0, exec_mode="warp")
        sa, sb = a.samples.cpu().numpy(), b.samples.cpu().numpy()
        assert np.isfinite(sb).all()
        assert close(sb[:, :2], sa[:, :2], BLOCK_REL, atol=BLOCK_REL)


def test_row_shard_exchange_emulated_ranks_bitwise():
    """The multi-GPU exchange device code with 2/4/8 ranks emulated as CTA
    groups of one launch (row shards, per-rank barriers and accumulators,
    mailbox push/flags/sum): the wide-p chain is bit-identical to the
    unsharded one, across launches."""
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(20005, 255, 21)
    base = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="fp32")
    cfg = t.RunConfig(model={}, num_chains=1, num_warmup=30, num_samples=20, seed=6)
    keys = t.chain_keys(6, 1)
    ref = t.run_device(base, cfg, keys, 0)
    q = np.random.default_rng(2).standard_normal((2, 256)) * 0.05
    ref_ug = t.models.potential_and_gradient(base.device_spec, q)
    for V in (2, 4, 8):
        m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="fp32")
        t.rowshard.emulate_ranks(m.device_spec, V)
        assert np.array_equal(t.models.potential_and_gradient(m.device_spec, q), ref_ug), V
        for _ in range(2):
            r = t.run_device(m, cfg, keys, 0)
            assert np.array_equal(r.samples.cpu().numpy(), ref.samples.cpu().numpy()), V
            assert np.array_equal(r.stats.cpu().numpy(), ref.stats.cpu().numpy()), V


# ----------------------------------------------------------------------------- dense mass adaptation (8(f) item 3)


def test_pooled_covariance_matches_numpy():
    """Device pooled covariance vs numpy (ddof 1) on a ragged D (not a tile
    multiple) and an odd row count; regularised shrinkage; bitwise determinism."""
    import torch

    t = ts()
    gen = np.random.default_rng(3)
    n, D = 4999, 150
    x = gen.standard_normal((n, D)) @ gen.standard_normal((D, D)) * 0.3 + gen.standard_normal(D)
    xd = torch.from_numpy(x).cuda()
    mean, cov = t.pooled_covariance(xd, regularize=False)
    ref = np.cov(x.T)
    assert close(mean.cpu().numpy(), x.mean(0), 1e-12, atol=1e-12)
    assert np.abs(cov.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.array_equal(cov.cpu().numpy(), cov.cpu().numpy().T)
    _, reg = t.pooled_covariance(xd.reshape(7, n // 7, D) if n % 7 == 0 else xd, regularize=True)
    want = (n / (n + 5.0)) * ref + (5.0 / (n + 5.0)) * 1e-3 * np.eye(D)
    assert np.abs(reg.cpu().numpy() - want).max() <= 1e-12 * np.abs(want).max()
    _, again = t.pooled_covariance(xd, regularize=True)
    assert torch.equal(reg, again)
    # (C, S, D) input pools over chains
    _, c3 = t.pooled_covariance(xd[:4998].reshape(2, 2499, D), regularize=False)
    assert np.abs(c3.cpu().numpy() - np.cov(x[:4998].T)).max() <= 1e-12 * np.abs(ref).max()


def test_dense_mass_adaptation_two_phase():
    """Pilot run -> pooled covariance of its draws -> dense inverse mass:
    the adapted M^-1 approximates the target covariance and the adapted run
    needs fewer leapfrogs per draw than the identity-mass pilot."""
    t = ts()
    D, C = 24, 64
    A = _spd(D, 9, cond=300.0)
    cov = np.linalg.inv(A)
    cfg = t.RunConfig(model={}, num_chains=C, num_warmup=200, num_samples=200, seed=5)
    model, inv_mass, final = t.run_dense_adapted(A, cfg, precision="fp64", device=0)
    assert model.params["dense_mass"]
    err = np.linalg.norm(inv_mass - cov) / np.linalg.norm(cov)
    assert err < 0.2, err
    pilot = t.run_device(t.dense_gaussian_model(A, precision="fp64"), cfg, t.chain_keys(5, C), 0)
    lf_pilot = pilot.stats.cpu().numpy()[:, 200:, 1].mean()
    lf_final = final.stats.cpu().numpy()[:, 200:, 1].mean()
    assert lf_final < 0.7 * lf_pilot, (lf_final, lf_pilot)
    flat = final.samples.cpu().numpy().reshape(-1, D)
    assert np.abs(np.cov(flat.T) - cov).max() <= 0.15 * np.abs(cov).max()


# ----------------------------------------------------------------------------- fp64 X storage ("fp64x")


@pytest.mark.parametrize("n,p", [(3000, 54), (1001, 7), (700, 63), (50, 1), (517, 100), (2000, 255)])
def test_fp64x_non_fp32_exact_data(n, p, oracle):
    """Data that are not fp32-exact are stored in fp64 (the reference keeps
    fp64 X, models.py:43-64): precision "fp64" selects the fp64-storage pass
    automatically and matches the fp64 oracle at 1e-10 relative."""
    t = ts()
    rng = np.random.default_rng(p)
    x = rng.standard_normal((n, p))  # not fp32-exact
    y = (rng.random(n) < 0.5).astype(np.float64)
    data = t.LogisticRegressionData(x, y)
    assert data.x.dtype == np.float64
    m = t.logistic_regression_model(data, precision="fp64")
    assert m.device_spec.precision == "fp64x"
    om = oracle.Model("logistic_regression", p + 1, x=x, y=y)
    for q in (np.zeros(p + 1), rng.standard_normal(p + 1) * 0.1):
        got = t.models.potential_and_gradient(m.device_spec, q[None, :])[0]
        U = om.potential(q.tolist())
        g = np.asarray(om.gradient(q.tolist()))
        assert close(got[0], U, FP64_REL)
        assert close(got[1:], g, FP64_REL, atol=FP64_REL * np.abs(g).max())
    # the fp32 policy rounds such data with a warning (stated tolerance)
    with pytest.warns(RuntimeWarning):
        t.logistic_regression_model(data, precision="fp32")


def test_fp64x_covtype_transitions_match_oracle(oracle):
    """fp64 X storage at the covtype shape: transitions of a device run re-run
    from its own states on the CPU oracle: identical integers, positions 1e-12."""
    t = ts()
    from tests_data import logistic_data

    x, y = logistic_data(581012, 54, 20191222)
    m = t.logistic_regression_model(t.LogisticRegressionData(x, y), precision="fp64x")
    W, S, seed = 120, 8, 1003
    cfg = t.RunConfig(model={}, num_chains=1, num_warmup=W, num_samples=S, seed=seed)
    key = t.chain_keys(seed, 1)[0]
    r = t.run_device(m, cfg, [key], 0)
    st = r.stats.cpu().numpy()[0]
    ad = r.adapt.cpu().numpy()[0]
    samples = r.samples.cpu().numpy()[0]
    step, inv = float(ad[1]), ad[2 + W:].copy()
    om = oracle.Model("logistic_regression", 55, x=x, y=y, fused_omp=True)
    for i in (1, 4, 7):
        q0 = samples[i - 1]
        U0, g0 = m.potential(q0), m.gradient(q0)
        dkey = key.fold(10 + W + i)
        oz, os_, _ = oracle.transition(oracle.Point(q0.tolist(), [0.0] * 55, U0, g0.tolist()), step, inv.tolist(), om,
                                       (dkey.hi, dkey.lo))
        assert (os_.depth, os_.leapfrogs) == (int(st[W + i, 0]), int(st[W + i, 1]))
        assert close(samples[i], oz.q, 1e-12, atol=1e-14)
