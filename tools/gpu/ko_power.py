"""Sustained (power-capped) per-call time of one la_fwd at [8, 16, 8192, 128] for the library given by
LA_B200_LIB: burst (first 50 calls after 3 s idle) and sustained (after ~2 s of back-to-back calls)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate
dev = torch.device("cuda", 0)
lam = ops.decay_tensor([decay_rate(h, 1, 16, 16) for h in range(1, 17)], 16, dev)
q, k, v = (torch.randn(8, 16, 8192, 128, device=dev, dtype=torch.bfloat16) for _ in range(3))
time.sleep(3)
times = []
t_end = time.time() + 2.5
while time.time() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        ops.la_forward(q, k, v, None, lam_dev=lam)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / 50)
print(f"{os.environ.get('LA_B200_LIB', 'default')}: burst {times[0]:.4f} ms sustained {sorted(times[-10:])[5]:.4f} ms")
