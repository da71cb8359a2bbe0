"""GLA core forward: fused (la_gla_core_fwd) vs two-step (la_gla_prologue + la_fwd) at [8, 8192, 2048]."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_17381_b200 import ops  # noqa: E402
from oracle.linattn_oracle import decay_rate  # noqa: E402

H, D = 16, 128


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


lam = ops.decay_tensor([decay_rate(h, 1, H, 16) for h in range(1, H + 1)], H, "cuda")
theta = torch.tensor([10000.0 ** (-2.0 * j / D) for j in range(D // 2)], dtype=torch.float64, device="cuda")
for b, n in ((8, 8192), (64, 1024)):
    qp, kp, v = (torch.randn(b, n, H * D, device="cuda").to(torch.bfloat16) for _ in range(3))
    for th in (theta, None):
        pro = t_ms(lambda: ops.gla_prologue(qp, kp, H, theta=th))
        q2, k2 = ops.gla_prologue(qp, kp, H, theta=th)
        core = t_ms(lambda: ops.la_forward(*(t.view(b, n, H, D) for t in (q2, k2, v)), None, lam_dev=lam, layout="bnhd"))
        fused = t_ms(lambda: ops.gla_core_forward(qp, kp, v, None, H, theta=th, lam_dev=lam))
        fnq = t_ms(lambda: ops.gla_core_forward(qp, kp, v, None, H, theta=th, lam_dev=lam, want_qk=False))
        print(f"[{b},{n},{H * D}] lrpe={th is not None}: prologue {pro:.4f} + core {core:.4f} = {pro + core:.4f} ms | "
              f"fused {fused:.4f} ms (x{(pro + core) / fused:.2f}) | fused no q/k {fnq:.4f} ms (x{(pro + core) / fnq:.2f})",
              flush=True)

# the backward: fused (la_gla_core_bwd) vs two-step (la_bwd + la_gla_prologue_bwd)
for b, n in ((8, 8192), (64, 1024)):
    qp, kp, v, da = (torch.randn(b, n, H * D, device="cuda").to(torch.bfloat16) for _ in range(4))
    for th in (theta, None):
        _, q, k = ops.gla_core_forward(qp, kp, v, None, H, theta=th, lam_dev=lam)

        def two_step():
            dq, dk, dv = ops.la_backward(*(t.view(b, n, H, D) for t in (q, k, v, da)), None, lam_dev=lam, layout="bnhd")
            ops.gla_prologue_backward(qp, kp, dq.view(b, n, -1), dk.view(b, n, -1), H, theta=th)

        t2 = t_ms(two_step)
        tf = t_ms(lambda: ops.gla_core_backward(qp, kp, q, k, v, da, None, H, theta=th, lam_dev=lam))
        print(f"bwd [{b},{n},{H * D}] lrpe={th is not None}: two-step {t2:.4f} ms | fused {tf:.4f} ms (x{t2 / tf:.2f})",
              flush=True)
