"""Head dims below 128: fwd+bwd timing of the tensor-core passes (zero-padded d = 128 tiles) vs the SIMT
passes, bf16 and fp32 (CUDA events).  Decides the default route for d < 128."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_17381_b200 import ops  # noqa: E402
from oracle.linattn_oracle import decay_rate  # noqa: E402
from tc32_time import time_it  # noqa: E402

cases = [(1, 4, 1024, 64), (8, 16, 8192, 64), (16, 32, 2048, 64), (8, 16, 8192, 32), (8, 16, 8192, 96)]
if os.environ.get("LA_NO_SIMT"):  # A/B of tensor-core variants: skip the slow SIMT arm, add d = 128
    cases.append((8, 16, 8192, 128))
dtypes = (torch.bfloat16,) if os.environ.get("LA_BF16_ONLY") else (torch.bfloat16, torch.float32)
for dtype in dtypes:
    for b, h, n, d in cases:
        lams = [decay_rate(j + 1, 1, h, h) for j in range(h)]
        q, k, v, do = (torch.randn(b, h, n, d, device="cuda", dtype=dtype) / d ** 0.5 for _ in range(4))
        line = []
        for backend in ("tcgen05",) if os.environ.get("LA_NO_SIMT") else ("tcgen05", "simt"):
            f = time_it(lambda: ops.la_forward(q, k, v, lams, backend=backend))
            g = time_it(lambda: ops.la_backward(q, k, v, do, lams, backend=backend), reps=3)
            line.append(f"{backend}: fwd {f:.3f} bwd {g:.3f} ms ({b * n / (f + g) / 1e3:.1f}M tok/s)")
        print(f"{str(dtype)[6:]} b={b} h={h} n={n} d={d}  " + "  |  ".join(line), flush=True)
