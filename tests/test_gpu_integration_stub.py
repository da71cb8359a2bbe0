"""The reference-side ctypes binding shown in INTEGRATION.md §2 is executed as written (library
path substituted) and checked against the oracle -- the documented stub cannot rot."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n(# linattn/b200.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its ctypes stub"
    return m.group(1).replace("/path/to/libla_b200.so", str(ROOT / "paper_2405_17381_b200" / "libla_b200.so"))


def test_stub_present_and_compiles():
    compile(_stub_source(), "INTEGRATION.md", "exec")


@pytest.mark.gpu
def test_stub_runs_and_matches_oracle():
    from oracle import linattn_oracle as orc
    from paper_2405_17381_b200.errors import DomainError, ShapeError
    from paper_2405_17381_b200.kernels import AttentionConfig

    ns = {"ShapeError": ShapeError, "DomainError": DomainError}
    exec(_stub_source(), ns)
    rng = np.random.default_rng(3)
    n, d = 77, 16
    q, k, v = (rng.uniform(0.05, 1.0, (n, d)) for _ in range(3))
    cfg = AttentionConfig(n=n, d=d, B=16, lam=0.9, precision="reference")
    o = ns["lightning_forward_decay"](q, k, v, cfg)
    want = orc.left_product_forward(q, k, v, 0.9)
    assert np.max(np.abs(o - want) / np.abs(want)) < 1e-10
