"""Shared test plumbing.

Markers: ``gpu`` = needs a B200 (run on the GPU box via ``pytest -m gpu``);
everything else runs on the CPU build container.
"""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@lru_cache(maxsize=1)
def golden() -> dict:
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def golden_cases():
    g = golden()
    return [tuple(c) for c in json.loads(bytes(g["meta/cases"]).decode())]


def golden_config1() -> dict:
    return json.loads(bytes(golden()["meta/config1"]).decode())


def case_inputs(n, d, seed, dist, count=4):
    """Same generator as tests/golden/make_golden.py:make_inputs."""
    rng = np.random.default_rng(seed)
    if dist == "pos":
        return [rng.uniform(0.05, 1.0, (n, d)) for _ in range(count)]
    return [rng.standard_normal((n, d)) for _ in range(count)]


def config1_inputs():
    c = golden_config1()
    rng = np.random.default_rng(c["seed"])
    shape = (c["batch"], c["H"], c["n"], c["d"])
    return [rng.uniform(0.05, 1.0, shape) for _ in range(4)]


def golden_array(key, like):
    """Compare-ready view of a stored golden array: returns (ref, got_view_fn)."""
    g = golden()
    if key in g:
        return g[key], lambda a: np.asarray(a, dtype=np.float64)
    rowsum, sample = g[key + "/rowsum"], g[key + "/sample"]
    idx = np.arange(0, like.size, 97)

    def view(a):
        a = np.asarray(a, dtype=np.float64)
        return np.concatenate([a.sum(axis=1), a.reshape(-1)[idx]])

    return np.concatenate([rowsum, sample]), view


@pytest.fixture(scope="session")
def gold():
    return golden()
