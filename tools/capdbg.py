import sys, faulthandler; faulthandler.enable(); sys.path.insert(0, ".")
import torch
from paper_2405_17381_b200 import ops
dev = torch.device("cuda", 0)
mode = sys.argv[1]
q, k, v = (torch.randn(4, 16, 128, device=dev, dtype=torch.bfloat16) for _ in range(3))
kv = torch.zeros(4, 16, 128, 128, device=dev)
lam = ops.decay_tensor([0.9] * 16, 16, dev)
for _ in range(3): ops.la_decode(q, k, v, None, kv, lam_dev=lam)
torch.cuda.synchronize()
print("warm ok", flush=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, capture_error_mode=mode):
    o = ops.la_decode(q, k, v, None, kv, lam_dev=lam)
print("captured", flush=True)
g.replay(); torch.cuda.synchronize(); print("replayed", flush=True)
