"""GLA stage kernels alone at [8, 8192, 2048] bf16 (LRPE on): prologue / prologue backward / epilogues."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_17381_b200 import ops  # noqa: E402


def t_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


H, D = 16, 128
theta = torch.tensor([10000.0 ** (-2.0 * j / D) for j in range(D // 2)], dtype=torch.float64, device="cuda")
qp, kp, a, u = (torch.randn(8, 8192, H * D, device="cuda").to(torch.bfloat16) for _ in range(4))
rb = qp.numel() * 2
for name, fn, rows in (("prologue", lambda: ops.gla_prologue(qp, kp, H, theta=theta), 4),
                       ("prologue_bwd", lambda: ops.gla_prologue_backward(qp, kp, a, u, H, theta=theta), 6),
                       ("prologue_bwd (no LRPE)", lambda: ops.gla_prologue_backward(qp, kp, a, u, H), 6)):
    ms = t_ms(fn)
    print(f"{name}: {ms:.4f} ms, {rows * rb / (ms / 1e3) / 1e9:.0f} GB/s", flush=True)
