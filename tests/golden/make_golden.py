"""Generate golden vectors by running the REAL reference package (linattn).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  The fixture is committed; the GPU box never
reads /root/reference.  Inputs are regenerated from the recorded seeds by
tests (numpy's default_rng/PCG64 stream is stable), so only outputs plus the
case table are stored.  For the config-1 shape (batch=1, H=4, n=1024, d=64)
only per-row sums and a strided sample of entries are stored to keep the
fixture small.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.npz"

# case table: (name, n, d, B, lam, seed, dist)
CASES = []
for n in (1, 2, 5, 31, 64, 257):
    for d in (1, 4, 16):
        for lam in (1.0, 0.9, 0.5):
            for B in sorted({1, 3, d, n}):
                CASES.append((f"grid_n{n}_d{d}_B{B}_l{lam}", n, d, B, lam, 1000 + n * 7 + d * 3 + B, "pos"))
# pinned points of the reference test-suite (test_kernels.py:103-110, 155-173)
CASES.append(("pinned_n64_d16_B8", 64, 16, 8, 0.8, 5, "pos"))
CASES.append(("pinned_n64_d16_B32", 64, 16, 32, 0.8, 5, "pos"))
CASES.append(("fp32_n65_d16_B16", 65, 16, 16, 0.9, 11, "pos"))
CASES.append(("mixed_n64_d16_l1", 64, 16, 16, 1.0, 10, "normal"))
CASES.append(("mixed_n64_d16_l09", 64, 16, 16, 0.9, 10, "normal"))
# tile-shaped cases matching the CUDA chunk sizes
for n, d, B, lam in ((300, 64, 64, 0.95), (300, 128, 128, 0.99), (513, 128, 64, 0.7), (129, 128, 128, 1.0)):
    CASES.append((f"tile_n{n}_d{d}_B{B}_l{lam}", n, d, B, lam, 77 + n + d, "pos"))

CONFIG1 = dict(batch=1, H=4, n=1024, d=64, B=64, lams=(1.0, 0.99, 0.9, 0.5), seed=2405)


def make_inputs(n, d, seed, dist, count=4):
    rng = np.random.default_rng(seed)
    if dist == "pos":
        return [rng.uniform(0.05, 1.0, (n, d)) for _ in range(count)]
    return [rng.standard_normal((n, d)) for _ in range(count)]


def config1_inputs():
    c = CONFIG1
    rng = np.random.default_rng(c["seed"])
    shape = (c["batch"], c["H"], c["n"], c["d"])
    return [rng.uniform(0.05, 1.0, shape) for _ in range(4)]


def sample_index(size: int) -> np.ndarray:
    return np.arange(0, size, 97)


def store(out, key, arr):
    """Full array when small, else per-row sums + a strided sample."""
    arr = np.asarray(arr)
    keep = np.float32 if arr.dtype == np.float32 else np.float64
    if arr.size <= 4096:
        out[key] = arr.astype(keep)
    else:
        a64 = arr.astype(np.float64)
        out[key + "/rowsum"] = a64.sum(axis=1)
        out[key + "/sample"] = a64.reshape(-1)[sample_index(a64.size)]


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    import linattn  # noqa: F401  (the reference)
    from linattn.kernels import AttentionConfig, lightning_backward_decay, lightning_forward_decay
    from linattn.matrixops import causal_decay_mask, decay_powers
    from linattn.oracles import left_product_forward, reference_backward
    from linattn.positional import decay_rate

    out: dict[str, np.ndarray] = {}
    for name, n, d, B, lam, seed, dist in CASES:
        q, k, v, do = make_inputs(n, d, seed, dist)
        c64 = AttentionConfig(n=n, d=d, B=B, lam=lam, precision="reference")
        c32 = AttentionConfig(n=n, d=d, B=B, lam=lam, precision="working")
        g = lightning_backward_decay(q, k, v, do, c64)
        g32 = lightning_backward_decay(q, k, v, do, c32)
        results = {
            "o64": lightning_forward_decay(q, k, v, c64),
            "dq64": g.dq, "dk64": g.dk, "dv64": g.dv,
            "o32": lightning_forward_decay(q, k, v, c32),
            "dq32": g32.dq, "dk32": g32.dk, "dv32": g32.dv,
        }
        if n * d <= 4096:  # the O(n^2)/per-token oracles only for small cases
            r = reference_backward(q, k, v, do, lam)
            results.update(left=left_product_forward(q, k, v, lam), rdq=r.dq, rdk=r.dk, rdv=r.dv)
        for key, arr in results.items():
            store(out, f"{name}/{key}", arr)

    # config 1 (BASELINE.json configs[0]): fp64 + fp32 reference outputs, compressed
    c = CONFIG1
    q, k, v, do = config1_inputs()
    for h, lam in enumerate(c["lams"]):
        for prec, tag in (("reference", "64"), ("working", "32")):
            cfg = AttentionConfig(n=c["n"], d=c["d"], B=c["B"], lam=lam, precision=prec)
            o = lightning_forward_decay(q[0, h], k[0, h], v[0, h], cfg)
            g = lightning_backward_decay(q[0, h], k[0, h], v[0, h], do[0, h], cfg)
            for key, arr in (("o", o), ("dq", g.dq), ("dk", g.dk), ("dv", g.dv)):
                arr = np.asarray(arr, dtype=np.float64)
                out[f"config1/h{h}/{key}{tag}/rowsum"] = arr.sum(axis=1)
                out[f"config1/h{h}/{key}{tag}/sample"] = arr.reshape(-1)[sample_index(arr.size)]

    # substrate known answers
    out["substrate/mask_7_0.6"] = causal_decay_mask(7, 0.6)
    out["substrate/powers_9_0.7_first1"] = decay_powers(9, 0.7, first=1)
    out["substrate/powers_9_0.7_first0"] = decay_powers(9, 0.7, first=0)
    table = np.array([[decay_rate(h, l, 16, 16) for l in range(1, 17)] for h in range(1, 17)])
    out["substrate/decay_rate_H16_L16"] = table

    out["meta/cases"] = np.frombuffer(json.dumps(CASES).encode(), dtype=np.uint8)
    out["meta/config1"] = np.frombuffer(json.dumps(CONFIG1).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **out)
    print(f"wrote {len(out)} arrays to {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
