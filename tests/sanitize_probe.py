# small fwd+bwd on both backends, for compute-sanitizer (memcheck / racecheck / synccheck)
import sys, torch
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops
for dtype, backend, n, segs in ((torch.bfloat16, "tcgen05", 300, 0), (torch.bfloat16, "tcgen05", 1000, 3),
                                (torch.float32, "simt", 100, 2)):
    q, k, v, do = (torch.rand(1, 2, n, 128, device="cuda", dtype=dtype) for _ in range(4))
    o, seg = ops.la_forward(q, k, v, [0.9, 0.99], backend=backend, segments=segs, want_seg_states=True)
    ops.la_backward(q, k, v, do, [0.9, 0.99], backend=backend, segments=segs, fwd_seg_states=seg)
torch.cuda.synchronize()
print("ok")
