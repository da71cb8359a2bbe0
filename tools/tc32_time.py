"""fp32 fwd+bwd timing at the TNL-1B shape: tensor-core split pass vs the SIMT pass (CUDA events)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_17381_b200 import ops  # noqa: E402
from oracle.linattn_oracle import decay_rate  # noqa: E402


def time_it(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    H = 16
    lams = [decay_rate(h + 1, 1, H, 16) for h in range(H)]
    for n, b in ((1024, 64), (8192, 8), (65536, 1)):
        q, k, v, do = (torch.randn(b, H, n, 128, device="cuda") / 128 ** 0.5 for _ in range(4))
        for backend in ("tcgen05", "simt"):
            if backend == "simt" and n > 8192:
                continue
            f = time_it(lambda: ops.la_forward(q, k, v, lams, backend=backend))
            g = time_it(lambda: ops.la_backward(q, k, v, do, lams, backend=backend), reps=3)
            print(f"n={n} b={b} {backend}: fwd {f:.3f} ms bwd {g:.3f} ms  {b * n / (f + g) / 1e3:.2f}M tok/s", flush=True)
