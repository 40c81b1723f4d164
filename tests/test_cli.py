"""CLI surface and run-output formats (reference tests/test_cli.py).

CPU tests: argument errors, exit codes and the CSV / JSON formats on
hand-built chain results.  GPU tests: the reference's CLI cases end to end
through the device sampler, plus chain sharding byte-stability.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from paper_1912_11554_b200 import cli
from paper_1912_11554_b200.chains import ChainResult, RunConfig
from paper_1912_11554_b200.diagnostics import summarize
from paper_1912_11554_b200.models import std_normal_model
from paper_1912_11554_b200.output import SCHEMA_VERSION, run_report, strip_timing, write_samples_csv


@pytest.fixture()
def model_file(tmp_path):
    path = tmp_path / "model.json"
    path.write_text(json.dumps({"model": "std_normal", "params": {"dim": 2}}))
    return path


def _fake_results(C=2, S=20, D=2, seed=0):
    gen = np.random.default_rng(seed)
    out = []
    for c in range(C):
        stats = np.column_stack([gen.integers(1, 5, S), gen.integers(1, 16, S), np.zeros(S),
                                 gen.random(S), gen.standard_normal(S)]).astype(np.float64)
        adaptation = {"initial_step_size": 1.0, "step_size_trace": [0.5] * 25, "final_step_size": 0.7,
                      "inv_mass_diag": [1.0] * D}
        out.append(ChainResult(c, gen.standard_normal((S, D)) / 3.0, stats, adaptation, 1234 + c,
                               int(stats[:, 1].sum()) + 100, int(stats[:, 1].sum())))
    return out


def test_bad_flags_exit_2():
    with pytest.raises(SystemExit) as err:
        cli.main(["sample", "--nonsense"])
    assert err.value.code == 2


def test_unknown_command_exit_2():
    with pytest.raises(SystemExit) as err:
        cli.main(["dance"])
    assert err.value.code == 2


def test_zero_warmup_without_step_size_exit_2(model_file):
    assert cli.main(["sample", "--model", str(model_file), "--warmup", "0", "--samples", "5"]) == 2


def test_unknown_extension_exit_2(model_file, tmp_path):
    assert cli.main(["sample", "--model", str(model_file), "--warmup", "25", "--samples", "5",
                     "--out", str(tmp_path / "draws.parquet")]) == 2


def test_csv_format_round_trips(tmp_path):
    results = _fake_results()
    path = tmp_path / "d.csv"
    write_samples_csv(path, results)
    lines = path.read_text().splitlines()
    assert lines[0] == "chain,dim_0,dim_1"
    assert len(lines) == 1 + 2 * 20
    rows = np.array([[float(v) for v in ln.split(",")[1:]] for ln in lines[1:]])
    assert np.array_equal(rows, np.concatenate([r.samples for r in results]))  # repr is exact
    assert [ln.split(",")[0] for ln in lines[1:]] == ["0"] * 20 + ["1"] * 20


def test_json_report_schema(tmp_path):
    results = _fake_results()
    model = std_normal_model(2)
    config = RunConfig(model=model.descriptor(), num_chains=2, num_warmup=25, num_samples=20, seed=3)
    doc = run_report(config, model, results, summarize(results), include_trace=True)
    doc = json.loads(json.dumps(doc))
    assert doc["schema_version"] == SCHEMA_VERSION == 1
    assert doc["model"]["model"] == "std_normal"
    assert doc["run"] == {"num_chains": 2, "num_warmup": 25, "num_samples": 20, "mode": "sequential", "seed": 3}
    assert len(doc["chains"]) == 2 and len(doc["chains"][0]["samples"]) == 20
    assert len(doc["chains"][0]["adaptation"]["step_size_trace"]) == 25
    assert {"mean", "std", "ess", "split_rhat"} <= set(doc["summary"])
    c0 = doc["chains"][0]
    assert c0["max_depth_reached"] == int(results[0].stats_array[:, 0].max())
    assert c0["mean_accept_stat"] == pytest.approx(results[0].stats_array[:, 3].mean())
    no_trace = run_report(config, model, results, summarize(results))
    assert "step_size_trace" not in no_trace["chains"][0]["adaptation"]
    stripped = strip_timing(doc)
    assert "elapsed_ns" not in stripped["summary"] and "elapsed_ns" not in stripped["chains"][0]
    assert "elapsed_ns" in doc["summary"]  # deep copy


@pytest.mark.gpu
def test_sample_writes_csv_byte_stable(model_file, tmp_path):
    args = ["sample", "--model", str(model_file), "--chains", "2", "--warmup", "25", "--samples", "20", "--seed", "3"]
    out, out2 = tmp_path / "draws.csv", tmp_path / "again.csv"
    assert cli.main(args + ["--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "chain,dim_0,dim_1" and len(lines) == 41 and lines[1].split(",")[0] == "0"
    assert cli.main(args + ["--out", str(out2)]) == 0
    assert out.read_bytes() == out2.read_bytes()


@pytest.mark.gpu
def test_sample_writes_versioned_json(model_file, tmp_path):
    out = tmp_path / "report.json"
    assert cli.main(["sample", "--model", str(model_file), "--chains", "2", "--warmup", "25", "--samples", "20",
                     "--seed", "3", "--out", str(out), "--adapt-trace"]) == 0
    doc = json.loads(out.read_text())
    assert doc["schema_version"] == 1 and doc["run"]["num_chains"] == 2
    assert len(doc["chains"]) == 2 and len(doc["chains"][0]["samples"]) == 20
    assert len(doc["chains"][0]["adaptation"]["step_size_trace"]) == 25


@pytest.mark.gpu
def test_sample_modes_and_layouts_agree_modulo_timing(model_file, tmp_path):
    docs = {}
    for mode in ("seq", "par"):
        out = tmp_path / f"{mode}.json"
        assert cli.main(["sample", "--model", str(model_file), "--chains", "3", "--warmup", "25", "--samples", "15",
                         "--seed", "11", "--mode", mode, "--out", str(out)]) == 0
        docs[mode] = strip_timing(json.loads(out.read_text()))
    for doc in docs.values():
        doc["run"].pop("mode")
    assert docs["seq"] == docs["par"]


@pytest.mark.gpu
def test_sample_zero_warmup_with_step_size(model_file):
    assert cli.main(["sample", "--model", str(model_file), "--warmup", "0", "--samples", "5",
                     "--step-size", "0.5"]) == 0


@pytest.mark.gpu
def test_compare_trees_passes_and_reports(capsys):
    assert cli.main(["compare-trees", "--depth-max", "4", "--trials", "6", "--seed", "7"]) == 0
    out = capsys.readouterr().out
    for depth in range(5):
        assert f"depth {depth}: 6/6" in out


@pytest.mark.gpu
def test_bench_reports(model_file, tmp_path, capsys):
    out = tmp_path / "bench.json"
    assert cli.main(["bench", "--model", str(model_file), "--warmup", "30", "--samples", "30",
                     "--tree-depth", "5", "--reps", "2", "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["builders"]["iterative"]["time_per_leapfrog_ns"] > 0
    assert set(doc["tree_microbench"]["ns_per_leapfrog"]) == {"thread", "block", "warp"}


def _close(a, b, rel):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and bool(np.allclose(a, b, rtol=rel, atol=rel, equal_nan=True))


@pytest.mark.gpu
def test_sample_outputs_match_reference_cli(tmp_path):
    """The reference CLI's own CSV and JSON report (tests/golden/cli.json,
    made by tests/golden/make_cli_golden.py) reproduced through our CLI:
    format, chain ids, per-chain integer statistics (leapfrogs, divergences,
    max depth) exact; draws and summary floats within 1e-10 (small models on
    the thread team are bit-identical up to last-ulp exp/log1p; the logistic
    fp64 pass differs in summation order only)."""
    from conftest import golden

    g = golden("cli")
    (tmp_path / "data.csv").write_text(g["data_csv"])
    for case in g["cases"]:
        mpath = tmp_path / "model.json"
        mpath.write_text(json.dumps(case["desc"]))
        base = ["sample", "--model", str(mpath)] + case["args"]
        assert cli.main(base + ["--out", str(tmp_path / "s.csv")]) == 0
        assert cli.main(base + ["--out", str(tmp_path / "r.json")]) == 0
        ours = (tmp_path / "s.csv").read_text().splitlines()
        ref = case["csv"].splitlines()
        assert ours[0] == ref[0] and len(ours) == len(ref), case["desc"]
        assert [ln.split(",")[0] for ln in ours] == [ln.split(",")[0] for ln in ref]
        assert _close([[float(v) for v in ln.split(",")[1:]] for ln in ours[1:]],
                      [[float(v) for v in ln.split(",")[1:]] for ln in ref[1:]], 1e-10), case["desc"]
        doc = strip_timing(json.loads((tmp_path / "r.json").read_text()))
        rdoc = case["report"]
        assert doc["schema_version"] == rdoc["schema_version"]
        assert doc["model"] == rdoc["model"] and doc["run"] == rdoc["run"]
        assert set(doc["summary"]) == set(rdoc["summary"])
        assert doc["summary"]["total_leapfrogs"] == rdoc["summary"]["total_leapfrogs"]
        assert doc["summary"]["divergences"] == rdoc["summary"]["divergences"]
        for k in ("mean", "std", "ess", "split_rhat"):
            assert _close(doc["summary"][k], rdoc["summary"][k], 1e-8), (case["desc"], k)
        for c, rc in zip(doc["chains"], rdoc["chains"], strict=True):
            assert set(c) == set(rc)
            for k in ("chain_id", "divergences", "total_leapfrogs", "sampling_leapfrogs", "max_depth_reached"):
                assert c[k] == rc[k], (case["desc"], k)
            assert _close(c["mean_accept_stat"], rc["mean_accept_stat"], 1e-10)
            assert _close(c["samples"], rc["samples"], 1e-10)
            assert c["adaptation"] == rc["adaptation"]


def test_cli_golden_fixture_is_consistent():
    """CPU check of the committed reference fixture: CSV rows and report
    samples agree, and the logistic data are fp32-exact."""
    from conftest import golden

    g = golden("cli")
    assert len(g["cases"]) == 4
    for case in g["cases"]:
        rows = case["csv"].splitlines()[1:]
        samples = [s for ch in case["report"]["chains"] for s in ch["samples"]]
        assert np.array_equal([[float(v) for v in ln.split(",")[1:]] for ln in rows], samples)
    for ln in g["data_csv"].splitlines()[1:]:
        x = [float(v) for v in ln.split(",")[:-1]]
        assert np.array_equal(np.float32(x).astype(np.float64), x)
