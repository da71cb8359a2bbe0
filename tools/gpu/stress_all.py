"""Soak test of every tensor-core path (bf16 / fp32, d = 32..128, split and unsplit sequences, states,
GLA core): random shapes for LA_STRESS_S seconds, each problem run twice and required to be bitwise
identical (the kernels are deterministic) and finite; every 10th problem also against the SIMT backend
(fp32 1e-4 / bf16 2e-2 relative on positive inputs).  Catches intermittent launch failures and races
that a single parity run can miss."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_17381_b200 import ops  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("LA_STRESS_SEED", "1")))
budget = float(os.environ.get("LA_STRESS_S", "240"))
t_end = time.time() + budget
done = checked = 0
while time.time() < t_end:
    dtype = [torch.bfloat16, torch.float32][rng.integers(2)]
    d = int(rng.choice([32, 64, 96, 128, 128, 128]))
    b, h = int(rng.integers(1, 9)), int(rng.choice([1, 2, 4, 16, 32]))
    n = int(rng.choice([1, 100, 128, 129, 1000, 4096, 8192, 20000]))
    while b * h * n * d > (1 << 26):
        b = max(1, b // 2) if b > 1 else b
        if b == 1:
            n = max(1, n // 2)
    segs = int(rng.choice([0, 0, 0, 2, 5]))
    lams = [float(rng.choice([1.0, 0.999, 0.99, 0.9, 0.5, 5.5e-4])) for _ in range(h)]
    q, k, v, do = (torch.rand(b, h, n, d, device="cuda", dtype=dtype) for _ in range(4))
    kv = torch.rand(b, h, d, d, device="cuda") * 0.01 if rng.random() < 0.5 else None
    outs = []
    for _ in range(2):
        (o, kvo), seg = ops.la_forward(q, k, v, lams, kv_in=kv, want_state=True, want_seg_states=True,
                                       backend="tcgen05", segments=segs)
        g = ops.la_backward(q, k, v, do, lams, kv_in=kv, backend="tcgen05", segments=segs, fwd_seg_states=seg)
        outs.append([o, kvo, *g])
    torch.cuda.synchronize()
    for a, c in zip(*outs):
        assert torch.equal(a, c), f"nondeterministic: {dtype} b={b} h={h} n={n} d={d} segs={segs}"
        assert torch.isfinite(a).all(), f"non-finite: {dtype} b={b} h={h} n={n} d={d} segs={segs}"
    if done % 10 == 0 and b * h * n <= (1 << 18):
        ref = [ops.la_forward(q, k, v, lams, kv_in=kv, backend="simt"),
               *ops.la_backward(q, k, v, do, lams, kv_in=kv, backend="simt")]
        got = [outs[0][0], *outs[0][2:]]
        tol = 2e-4 if dtype == torch.float32 else 4e-2
        for a, r in zip(got, ref):
            err = ((a.double() - r.double()).abs() / r.double().abs().clamp_min(1e-6)).max().item()
            assert err <= tol, f"tc vs simt {err:.3e}: {dtype} b={b} h={h} n={n} d={d} segs={segs}"
        checked += 1
    done += 1
# the fused GLA core (bf16, d = 128), split and unsplit
theta = torch.rand(64, dtype=torch.float64, device="cuda")
for b, n, hh in ((8, 1024, 16), (1, 9000, 4)):
    qp, kp, v, da = (torch.rand(b, n, hh * 128, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    lam = [0.9, 0.99, 0.5, 1.0] * (hh // 4)
    r1 = ops.gla_core_forward(qp, kp, v, lam, hh, theta=theta, offset=3)
    r2 = ops.gla_core_forward(qp, kp, v, lam, hh, theta=theta, offset=3)
    assert all(torch.equal(x, y) for x, y in zip(r1, r2))
torch.cuda.synchronize()
print(f"stress ok: {done} problems ({checked} checked against SIMT) in {budget:.0f} s")
