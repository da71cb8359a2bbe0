import sys; sys.path.insert(0, '.')
import torch
from paper_2405_17381_b200 import ops
from oracle.linattn_oracle import decay_rate
lams = [decay_rate(h + 1, 1, 16, 16) for h in range(16)]
for n, b in ((1024, 64), (8192, 8), (65536, 1)):
    q, k, v, do = (torch.randn(b, 16, n, 128, device="cuda") / 128 ** 0.5 for _ in range(4))
    for it in range(3):
        ops.la_forward(q, k, v, lams); torch.cuda.synchronize()
        print("fwd ok", n, it, flush=True)
        ops.la_backward(q, k, v, do, lams); torch.cuda.synchronize()
        print("bwd ok", n, it, flush=True)
