"""Pin the CPU oracle against the reference's own outputs (tests/golden).

The golden fixtures were produced by running the unmodified reference
(turnstile, numba path) in the build container; see tests/golden/make_golden.py.
Small-model results must agree BIT FOR BIT (the oracle keeps the reference's
operation order); logistic results go through oracle/logistic_ref.c, whose
sequential loop also reproduces the numba path exactly.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden, num, nums


def test_philox_and_key_derivation(oracle):
    for rec in golden("rng")["seeds"]:
        seed = int(rec["seed"])
        key = oracle.key_from_seed(seed)
        assert [str(key[0]), str(key[1])] == rec["key"]
        a, b = oracle.key_split(key)
        assert [[str(a[0]), str(a[1])], [str(b[0]), str(b[1])]] == rec["split"]
        for i, words in rec["fold"].items():
            k = oracle.key_fold(key, int(i))
            assert [str(k[0]), str(k[1])] == words


def test_uniform_and_normal_streams(oracle):
    for rec in golden("rng")["seeds"][:3]:
        key = (int(rec["key"][0]), int(rec["key"][1]))
        s = oracle.Stream(key)
        assert [s.random() for _ in range(70)] == nums(rec["uniform"])
        s = oracle.Stream(key)
        assert [s.normal() for _ in range(300)] == nums(rec["normal"])
        s = oracle.Stream(key)
        assert [-2.0 + 4.0 * s.random() for _ in range(9)] == nums(rec["uniform_m2_2"])


def test_normals_against_numpy_many(oracle):
    """The restated ziggurat equals numpy's Generator.standard_normal, tails included."""
    from numpy.random import Generator, Philox

    key = (0x1234567890ABCDEF, 0x0FEDCBA987654321)
    g = Generator(Philox(counter=np.array([0, 0, 0, 1], dtype=np.uint64), key=np.array(key, dtype=np.uint64)))
    ref = g.standard_normal(40000)
    s = oracle.Stream(key)
    got = np.array([s.normal() for _ in range(40000)])
    assert np.array_equal(got, ref)
    assert np.abs(ref).max() > 3.6541528853610088  # the tail branch was exercised


def _tree_case(oracle, case):
    m = oracle.model_from_desc(case["model"])
    z = oracle.Point(nums(case["z"]["q"]), nums(case["z"]["r"]), num(case["z"]["U"]), nums(case["z"]["g"]))
    key = (int(case["key"][0]), int(case["key"][1]))
    return oracle.build_tree(z, case["depth"], num(case["eps"]), nums(case["inv_diag"]), m, key, num(case["h_ref"]),
                             case["criterion"] == "generalized", num(case["threshold"]))


def test_tree_battery_bitwise(oracle):
    for i, case in enumerate(golden("trees")):
        t = _tree_case(oracle, case)
        o = case["out"]
        assert t.sub.count == o["leapfrog_count"], i
        assert t.turning == o["turning"] and t.diverging == o["diverging"], i
        assert t.sub.prop_leaf == o["proposal_leaf"], i
        assert [list(w) for w in t.writes] == case["trace"]["writes"], i
        assert [list(c) for c in t.checks] == case["trace"]["checks"], i
        assert t.max_occupied == case["trace"]["max_occupied"], i
        assert t.sub.lw == num(o["log_weight"]) or (math.isinf(t.sub.lw) and o["log_weight"] == "-inf"), i
        assert t.sub.metro == num(o["sum_metropolis"]), i
        assert t.msum == nums(o["momentum_sum"]), i
        assert t.sub.last.q == nums(o["right_q"]) and t.sub.last.r == nums(o["right_r"]), i
        assert t.sub.first.q == nums(o["left_q"]) and t.sub.first.r == nums(o["left_r"]), i
        assert t.sub.prop.q == nums(o["prop_q"]) and t.sub.prop.U == num(o["prop_U"]), i
        assert t.leaf_lw == nums(case["trace"]["leaf_log_weights"]), i


def test_schedule_kats(oracle):
    """Reference KATs: step 11 checks (slot 2, leaf 10) then (slot 1, leaf 8);
    depth-2 schedule writes [(0,0),(2,1)] checks [(1,0),(3,1),(3,0)]."""
    case = [c for c in golden("trees") if c["depth"] == 4 and c["eps"] == 1e-3][0]
    t = _tree_case(oracle, case)
    assert [(s, leaf) for n, s, leaf in t.checks if n == 11] == [(2, 10), (1, 8)]
    m = oracle.Model("std_normal", 2)
    g = oracle.Stream(oracle.key_fold(oracle.key_from_seed(7), 0))
    q = [g.normal() * 0.5 for _ in range(2)]
    r = [g.normal() for _ in range(2)]
    z = oracle.Point(q, r, m.potential(q), m.gradient(q))
    t = oracle.build_tree(z, 2, 1e-3, [1.0, 1.0], m, oracle.key_from_seed(7), oracle.hamiltonian(z.U, z.r, [1, 1]))
    assert t.writes == [(0, 0), (2, 1)]
    assert [(n, s) for n, s, _ in t.checks] == [(1, 0), (3, 1), (3, 0)]


def test_transitions_bitwise(oracle):
    for rec in golden("transitions"):
        m = oracle.model_from_desc(rec["model"])
        inv = nums(rec["inv_diag"])
        for d in rec["draws"]:
            z = oracle.Point(nums(d["z_in"]["q"]), [0.0] * m.dim, num(d["z_in"]["U"]), nums(d["z_in"]["g"]))
            key = (int(d["key"][0]), int(d["key"][1]))
            z1, st, dec = oracle.transition(z, rec["step"], inv, m, key, rec["max_tree_depth"],
                                            rec["criterion"] == "generalized")
            assert [st.depth, st.leapfrogs, int(st.diverged)] == d["stats"][:3]
            assert st.accept == num(d["stats"][3]) and st.energy == num(d["stats"][4])
            assert [list(t) for t in dec["trees"]] == d["trees"]
            assert dec["outer"] == d["outer"]
            assert z1.q == nums(d["z_out"]["q"]) and z1.U == num(d["z_out"]["U"])


@pytest.mark.parametrize("idx", range(6))
def test_runs_bitwise(oracle, idx):
    rec = golden("runs")[idx]
    desc = rec["desc"]
    name = desc["model"]
    md = {"name": name, **desc["params"]}
    if name == "gaussian":
        md["cov_diag"] = desc["params"]["cov_diag"]
    m = oracle.model_from_desc(md)
    keys = oracle.chain_keys(rec["seed"], rec["num_chains"])
    s = rec["sampler"]
    for c, ref in enumerate(rec["chains"]):
        if s is None:
            out = oracle.run_chain(m, keys[c], rec["num_warmup"], rec["num_samples"])
        else:
            out = oracle.run_chain(m, keys[c], rec["num_warmup"], rec["num_samples"], step=s["step"], has_sampler=True,
                                   max_depth=s["max_tree_depth"], generalized=s["criterion"] == "generalized")
        assert out["total_leapfrogs"] == ref["total_leapfrogs"]
        got_stats = [[st.depth, st.leapfrogs, int(st.diverged), st.accept, st.energy] for st in out["stats"]]
        W = rec["num_warmup"]
        assert got_stats[W:] == [[v if isinstance(v, int) else num(v) for v in row] for row in ref["stats"]]
        assert out["samples"] == [nums(r) for r in ref["samples"]]
        assert out["adaptation"]["final_step_size"] == num(ref["adaptation"]["final_step_size"])


def test_logistic_c_oracle_matches_reference_numba(oracle):
    """oracle/logistic_ref.c (sequential) == turnstile numba kernels, bit for bit."""
    from tests_data import logistic_data

    for rec in golden("logistic"):
        x, y = logistic_data(rec["n"], rec["p"], rec["seed"])
        m = oracle.Model("logistic_regression", rec["p"] + 1, x=np.ascontiguousarray(x), y=np.ascontiguousarray(y))
        for p in rec["points"]:
            q = nums(p["q"])
            assert m.potential(q) == num(p["U"])
            assert m.gradient(q) == nums(p["g"])


def test_logistic_omp_close_to_sequential(oracle):
    import ctypes

    from tests_data import logistic_data

    x, y = logistic_data(20000, 54, 3)
    m = oracle.Model("logistic_regression", 55, x=np.ascontiguousarray(x), y=np.ascontiguousarray(y))
    q = np.random.default_rng(0).standard_normal(55) * 0.1
    out = np.zeros(56)
    x32 = np.ascontiguousarray(x, dtype=np.float32)
    y8 = np.ascontiguousarray(y, dtype=np.uint8)
    m.clib().ts_oracle_logistic_omp(x32.ctypes.data, y8.ctypes.data, 20000, 54, q.ctypes.data, out.ctypes.data)
    U = m.potential(q.tolist())
    g = np.asarray(m.gradient(q.tolist()))
    assert abs(out[0] - U) <= 1e-10 * abs(U)
    assert np.allclose(out[1:], g, rtol=1e-9, atol=1e-9)


def test_hmc_golden_bitwise(oracle):
    """Oracle restatement of sampler.hmc_transition vs the reference's own draws."""
    for case in golden("hmc"):
        m = oracle.model_from_desc(case["model"])
        inv = [1.0] * m.dim
        for d in case["draws"]:
            key = (int(d["key"][0]), int(d["key"][1]))
            q, st, _ = oracle.hmc_transition(nums(d["q_in"]), num(case["step"]), inv, m, key, case["num_steps"])
            assert q == nums(d["q_out"])
            assert st.leapfrogs == d["leapfrogs"] and st.diverged == d["diverged"]
            assert st.accept == num(d["accept_stat"]) and st.energy == num(d["energy"])
