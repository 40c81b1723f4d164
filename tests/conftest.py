"""Shared fixtures: the `gpu` marker, golden fixtures, the oracle module."""

from __future__ import annotations

import json
import math
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity against the oracle/golden data")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def num(x):
    """Decode the JSON float encoding of tests/golden (inf/nan as strings)."""
    if isinstance(x, str):
        return {"inf": math.inf, "-inf": -math.inf, "nan": math.nan}[x] if x in ("inf", "-inf", "nan") else float(x)
    return float(x)


def nums(xs):
    return [num(v) for v in xs]


_cache: dict = {}


def golden(name):
    if name not in _cache:
        with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
            _cache[name] = json.load(fh)
    return _cache[name]


@pytest.fixture(scope="session")
def oracle():
    import turnstile_oracle

    return turnstile_oracle
