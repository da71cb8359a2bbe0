"""Device timeline of one la_forward + la_backward (warm) per shape, from CUPTI via torch.profiler:
each kernel's start offset, duration and the idle gap before it.  A design probe, not a bench.

usage: python tools/timeline.py [b:n ...]   (default 8:8192 4:16384 2:32768 1:65536 1:131072)
       TL_H / TL_D / TL_DTYPE (bf16 | f32 | f64) set heads, head dim and dtype (default 16, 128, bf16)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate

dev = torch.device("cuda", 0)
H, D = int(os.environ.get("TL_H", 16)), int(os.environ.get("TL_D", 128))
DT = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[os.environ.get("TL_DTYPE", "bf16")]
lam = ops.decay_tensor([decay_rate(h, 1, H, 16) for h in range(1, H + 1)], H, dev)
shapes = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]] or [(8, 8192), (4, 16384), (2, 32768),
                                                                          (1, 65536), (1, 131072)]
for b, n in shapes:
    q, k, v, do = (torch.randn(b, H, n, D, device=dev, dtype=DT) * D ** -0.5 for _ in range(4))

    def fb():
        _, seg = ops.la_forward(q, k, v, None, lam_dev=lam, want_seg_states=True)
        ops.la_backward(q, k, v, do, None, lam_dev=lam, fwd_seg_states=seg)

    for _ in range(5):
        fb()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            fb()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    # the last iteration: from the last forward summary / pass launch group
    names = [e.name for e in evs]
    per_iter = len(evs) // 3
    it = evs[-per_iter:]
    t0 = it[0].time_range.start
    print(f"== b={b} n={n}: {per_iter} kernels, span {(it[-1].time_range.end - t0) / 1000:.4f} ms")
    prev_end = t0
    for e in it:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        print(f"  +{(s - t0) / 1000:8.4f} ms  dur {d / 1000:8.4f}  gap {(s - prev_end) / 1000:+8.4f}  "
              f"stream {getattr(e, 'device_index', 0)}  {e.name[:70]}")
        prev_end = max(prev_end, e.time_range.end)
