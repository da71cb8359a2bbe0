import os, sys, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_2405_17381_b200 import ops
dev = torch.device("cuda", 0)
kv = torch.zeros(8, 2, 128, 128, device=dev)
qd, kd, vd = (torch.randn(8, 2, 128, device=dev, dtype=torch.bfloat16) for _ in range(3))
lam = [0.9, 0.99]
for _ in range(50): ops.la_decode(qd, kd, vd, lam, kv)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(2000): ops.la_decode(qd, kd, vd, lam, kv)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
