# racecheck / memcheck probe of the fp32 split pass alone (la_tc32.cu): full and state-only modes
import sys, torch
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops
for n, segs in ((300, 0), (1000, 3)):
    q, k, v, do = (torch.rand(1, 2, n, 128, device="cuda", dtype=torch.float32) for _ in range(4))
    o, seg = ops.la_forward(q, k, v, [0.9, 0.99], backend="tcgen05", segments=segs, want_seg_states=True)
    ops.la_backward(q, k, v, do, [0.9, 0.99], backend="tcgen05", segments=segs, fwd_seg_states=seg)
torch.cuda.synchronize()
print("ok")
