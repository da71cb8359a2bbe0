"""Bench sweeps in bursts separated by idle gaps: does the per-step slowdown inside a run recover after a
pause (thermal / power) or not (allocator / address effects)?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate
dev = torch.device("cuda", 0)
H, D, TOK = 16, 128, 65536
lam = ops.decay_tensor([decay_rate(h, 1, H, 16) for h in range(1, H + 1)], H, dev)
ns = [1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072]
inp = {n: [torch.randn(max(1, TOK // n), H, n, D, device=dev, dtype=torch.bfloat16) for _ in range(4)] for n in ns}
def step():
    for n in ns:
        q, k, v, do = inp[n]
        _, seg = ops.la_forward(q, k, v, None, lam_dev=lam, want_seg_states=True)
        ops.la_backward(q, k, v, do, None, lam_dev=lam, fwd_seg_states=seg)
for _ in range(3): step()
torch.cuda.synchronize()
for burst, gap in ((0, 0.0), (1, 3.0), (2, 0.0), (3, 10.0)):
    time.sleep(gap)
    out = []
    for s in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); step(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    print(f"burst {burst} after {gap}s idle: " + " ".join(f"{x:.2f}" for x in out), flush=True)
