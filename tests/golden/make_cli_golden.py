"""Generate tests/golden/cli.json by running the REFERENCE CLI in this container.

Usage (from the repo root, where /root/reference exists):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_cli_golden.py

For each case, ``turnstile sample`` (reference cli.py:85-126) is run twice:
once writing the samples CSV (output.py:22-29) and once the schema-1 JSON
report (output.py:50-63, wall-clock fields removed with strip_timing).  The
cases use ``--warmup 0`` and a fixed ``--step-size`` so the whole chain is
reproduced by the device (with warmup, dual averaging amplifies last-ulp
exp() differences; see tests/test_gpu_parity.py::test_runs_match_reference).
The logistic case writes its 20-row data CSV from fixed numbers that are
also stored in the fixture.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numpy as np  # noqa: E402

from turnstile import cli  # noqa: E402
from turnstile.output import strip_timing  # noqa: E402

OUT = Path(__file__).resolve().parent / "cli.json"


def logistic_csv() -> str:
    gen = np.random.default_rng(5)
    rows = ["x0,x1,label"]
    for _ in range(20):
        x0, x1 = gen.standard_normal(2)
        # fp32-exact covariates: the device streams X in fp32 (models.py logistic_regression_model)
        rows.append(f"{float(np.float32(x0))!r},{float(np.float32(x1))!r},{int(gen.random() < 0.5)}")
    return "\n".join(rows) + "\n"


CASES = [
    {"desc": {"model": "std_normal", "params": {"dim": 3}},
     "args": ["--chains", "2", "--warmup", "0", "--samples", "30", "--seed", "3", "--step-size", "0.6"]},
    {"desc": {"model": "gaussian", "params": {"cov_diag": [2.0, 0.5]}},
     "args": ["--chains", "3", "--warmup", "0", "--samples", "20", "--seed", "9", "--step-size", "0.4",
              "--criterion", "classic", "--max-depth", "6"]},
    {"desc": {"model": "funnel", "params": {"dim": 3}},
     "args": ["--chains", "2", "--warmup", "0", "--samples", "25", "--seed", "99", "--step-size", "0.3"]},
    {"desc": {"model": "logistic_regression", "data_path": "data.csv"},
     "args": ["--chains", "2", "--warmup", "0", "--samples", "20", "--seed", "4", "--step-size", "0.25"]},
]


def main() -> None:
    data = logistic_csv()
    out = {"data_csv": data, "cases": []}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        (tmp / "data.csv").write_text(data)
        for case in CASES:
            mpath = tmp / "model.json"
            mpath.write_text(json.dumps(case["desc"]))
            base = ["sample", "--model", str(mpath)] + case["args"]
            assert cli.main(base + ["--out", str(tmp / "s.csv")]) == 0
            assert cli.main(base + ["--out", str(tmp / "r.json")]) == 0
            report = strip_timing(json.loads((tmp / "r.json").read_text()))
            out["cases"].append({"desc": case["desc"], "args": case["args"],
                                 "csv": (tmp / "s.csv").read_text(), "report": report})
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
