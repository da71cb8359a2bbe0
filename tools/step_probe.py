"""Per-step durations of the bench sweep (fwd+bwd at each n), to see run-to-run spread inside one run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate
dev = torch.device("cuda", 0)
H, D, TOK = 16, 128, 65536
lam = ops.decay_tensor([decay_rate(h, 1, H, 16) for h in range(1, H + 1)], H, dev)
ns = [1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072]
inp = {n: [torch.randn(max(1, TOK // n), H, n, D, device=dev, dtype=torch.bfloat16) for _ in range(4)] for n in ns}
def step(ev=None):
    for i, n in enumerate(ns):
        q, k, v, do = inp[n]
        if ev: ev[i].record()
        _, seg = ops.la_forward(q, k, v, None, lam_dev=lam, want_seg_states=True)
        ops.la_backward(q, k, v, do, None, lam_dev=lam, fwd_seg_states=seg)
    if ev: ev[len(ns)].record()
for _ in range(3): step()
torch.cuda.synchronize()
for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(ns) + 1)]
    step(ev)
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ns))]
    print(f"step {s}: total {ev[0].elapsed_time(ev[-1]):.3f} ms  " + " ".join(f"{p:.3f}" for p in per))
