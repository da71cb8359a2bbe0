# fwd+bwd time vs forced segment count at the long-n bench shapes (planner calibration)
import sys, torch, json
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate
dev = torch.device('cuda', 0)
lam = ops.decay_tensor([decay_rate(h, 1, 16, 16) for h in range(1, 17)], 16, dev)
res = {}
for n in (8192, 16384, 32768, 65536, 131072):
    b = max(1, 65536 // n)
    q, k, v, do = (torch.randn(b, 16, n, 128, device=dev, dtype=torch.bfloat16) * 0.1 for _ in range(4))
    auto = ops.segment_count(ops._desc(ops._geometry(q, "bhnd"), q.dtype, None, "auto", 0))
    for segs in sorted({1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 16, 18, 20, 24, 28, 32, 37, auto}):
        if segs > 592 // (b * 16) + 1:
            continue
        def step():
            o, seg = ops.la_forward(q, k, v, None, lam_dev=lam, segments=segs, want_seg_states=True)
            ops.la_backward(q, k, v, do, None, lam_dev=lam, segments=segs, fwd_seg_states=seg)
        for _ in range(2): step()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(5): step()
        e.record(); e.synchronize()
        ms = a.elapsed_time(e) / 5
        res.setdefault(n, {})[segs] = round(b * n / ms / 1e3, 1)  # M tokens/s
    best = max(res[n], key=res[n].get)
    print(n, "auto", auto, res[n][auto], "best", best, res[n][best], res[n], flush=True)
