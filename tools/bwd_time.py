"""bf16 backward timing over the bench's shapes (CUDA events): la_backward, and the dK/dV sweep alone
(parts="dkdv").  For same-box A/B of library variants (LA_B200_LIB)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_17381_b200 import ops  # noqa: E402
from oracle.linattn_oracle import decay_rate  # noqa: E402
from tc32_time import time_it  # noqa: E402

H = 16
lams = [decay_rate(h + 1, 1, H, 16) for h in range(H)]
line = []
for n, b in ((1024, 64), (8192, 8), (65536, 1)):
    q, k, v, do = (torch.randn(b, H, n, 128, device="cuda", dtype=torch.bfloat16) / 128 ** 0.5 for _ in range(4))
    g = time_it(lambda: ops.la_backward(q, k, v, do, lams), reps=20)
    s = time_it(lambda: ops.la_backward(q, k, v, do, lams, parts="dkdv"), reps=20)
    line.append(f"n={n}: bwd {g:.4f} dkdv {s:.4f}")
print("  ".join(line), flush=True)
