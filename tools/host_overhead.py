"""Host-side cost per call of the public entry points at a tiny shape (device work ~us): the floor a
launch-bound caller sees without CUDA graphs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17381_b200 import ops

dev = torch.device("cuda", 0)
q, k, v, do = (torch.randn(1, 2, 128, 128, device=dev, dtype=torch.bfloat16) for _ in range(4))
lam = [0.9, 0.99]
kv = torch.zeros(8, 2, 128, 128, device=dev)
qd, kd, vd = (torch.randn(8, 2, 128, device=dev, dtype=torch.bfloat16) for _ in range(3))
for name, fn in (("la_forward", lambda: ops.la_forward(q, k, v, lam)),
                 ("la_backward", lambda: ops.la_backward(q, k, v, do, lam)),
                 ("la_decode", lambda: ops.la_decode(qd, kd, vd, lam, kv))):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(1000):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host {1e6 * (t1 - t0) / 1000:.1f} us/call, wall {1e6 * (t2 - t0) / 1000:.1f} us/call")
