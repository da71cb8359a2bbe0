"""Per-kernel timing probe for design experiments (not a bench): la_forward and la_backward at a few
shapes, forced segment counts, CUDA events, median of reps.  LA_B200_LIB selects a library variant."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate

dev = torch.device("cuda", 0)
H, D = 16, 128
lams = [decay_rate(h, 1, H, 16) for h in range(1, H + 1)] if os.environ.get("LAMS", "bench") == "bench" else [0.99] * H
cases = [(8, 8192, 0), (1, 32768, 1), (4, 16384, 0), (1, 131072, 0)]
out = {}
for b, n, seg in cases:
    q, k, v, do = (torch.randn(b, H, n, D, device=dev, dtype=torch.bfloat16) * D ** -0.5 for _ in range(4))
    res = {}
    _, fst = ops.la_forward(q, k, v, lams, segments=seg, want_seg_states=True)
    for name, fn in (("fwd", lambda: ops.la_forward(q, k, v, lams, segments=seg, want_seg_states=True)),
                     ("bwd", lambda: ops.la_backward(q, k, v, do, lams, segments=seg, fwd_seg_states=fst))):
        for _ in range(3): fn()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        res[name] = round(sorted(ts)[len(ts) // 2], 4)
    out[f"{b}x{n}s{seg}"] = res
print(json.dumps(out))
