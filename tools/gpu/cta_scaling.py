"""Per-CTA chunk period of the dK/dV sweep and the dq pass vs the number of CTAs in flight (one wave,
unsplit sequences): does a CTA run faster when fewer CTAs share HBM?  [b, 16, 8192, 128] bf16."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_2405_17381_b200 import ops  # noqa: E402
from paper_2405_17381_b200.positional import decay_rate  # noqa: E402

dev = torch.device("cuda", 0)
lam = ops.decay_tensor([decay_rate(h, 1, 16, 16) for h in range(1, 17)], 16, dev)


def t_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n = 8192
for bsz in (1, 2, 4, 6, 8, 9):
    q, k, v, do = (torch.randn(bsz, 16, n, 128, device=dev).to(torch.bfloat16) for _ in range(4))
    kw = dict(lam_dev=lam, segments=1)
    t_f = t_ms(lambda: ops.la_forward(q, k, v, None, **kw))
    t_dq = t_ms(lambda: ops.la_backward(q, k, v, do, None, parts="dq", **kw))
    t_kv = t_ms(lambda: ops.la_backward(q, k, v, do, None, parts="dkdv", **kw))
    t_all = t_ms(lambda: ops.la_backward(q, k, v, do, None, **kw))
    ctas = bsz * 16
    chunks = n // 128
    cyc = lambda t: t * 1e-3 / chunks * 1.9e9  # noqa: E731  (cycles per chunk at ~1.9 GHz)
    gbs = lambda t, rows: bsz * 16 * n * rows * 256 / (t * 1e-3) / 1e9  # noqa: E731
    print(f"CTAs {ctas:4d}: fwd {t_f:.3f} ms ({cyc(t_f):.0f} cyc/chunk, {gbs(t_f, 4):.0f} GB/s)  "
          f"dq {t_dq:.3f} ({cyc(t_dq):.0f}, {gbs(t_dq, 4):.0f})  dkdv {t_kv:.3f} ({cyc(t_kv):.0f}, {gbs(t_kv, 6):.0f})  "
          f"bwd {t_all:.3f} ({gbs(t_all, 10):.0f} GB/s)", flush=True)
    del q, k, v, do
