"""Why the pass kernel is slower inside the bench sweep than timed alone: one la_fwd at [8, 16, 8192, 128]
timed (CUDA events, mean of 10) after different predecessors on the stream."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_17381_b200 import ops  # noqa: E402
from oracle.linattn_oracle import decay_rate  # noqa: E402

H = 16
lam = ops.decay_tensor([decay_rate(h + 1, 1, H, 16) for h in range(H)], H, "cuda")
mk = lambda b, n: [torch.randn(b, H, n, 128, device="cuda", dtype=torch.bfloat16) for _ in range(4)]  # noqa: E731
x8, x4 = mk(8, 8192), mk(16, 4096)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()


def timed(before, reps=10):
    for _ in range(3):
        before()
        ops.la_forward(*x8[:3], None, lam_dev=lam)
    ms = []
    for _ in range(reps):
        before()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ops.la_forward(*x8[:3], None, lam_dev=lam)
        b.record(stream)
        ms.append((a, b))
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in ms)


cases = {
    "after la_fwd (alone loop)": lambda: None,
    "after la_bwd at n=4096 (the sweep's order)": lambda: ops.la_backward(*x4, None, lam_dev=lam),
    "after a 512 MB memset (dirty L2)": lambda: flush.fill_(1),
    "after a 512 MB read (clean L2)": lambda: flush.sum(),
    "after host sync (idle GPU)": lambda: torch.cuda.synchronize(),
}
for name, fn in cases.items():
    print(f"{name:45s} {timed(fn):.4f} ms", flush=True)
