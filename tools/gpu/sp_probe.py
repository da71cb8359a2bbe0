"""Time the sequence-parallel path at one rank against the plain entry points (512K / 1M tokens, TNL-1B)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_2405_17381_b200 import ops, sp  # noqa: E402
from paper_2405_17381_b200.positional import decay_rate  # noqa: E402

dev = torch.device("cuda", 0)
H, D = 16, 128
lam = ops.decay_tensor([decay_rate(h, 1, H, 16) for h in range(1, H + 1)], H, dev)
g = torch.Generator(device=dev).manual_seed(0)


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for n in (524288, 1048576, 524288):
    q, k, v, do = ((torch.randn(1, H, n, D, device=dev, generator=g) / D ** 0.5).to(torch.bfloat16) for _ in range(4))
    leaves = [t.detach().clone().requires_grad_(True) for t in (q, k, v)]

    def plain():
        _, seg = ops.la_forward(q, k, v, None, lam_dev=lam, want_seg_states=True)
        ops.la_backward(q, k, v, do, None, lam_dev=lam, fwd_seg_states=seg)

    def plain_fwd():
        ops.la_forward(q, k, v, None, lam_dev=lam, want_seg_states=True)

    def sp_fb():
        o = sp.sp_lightning_attention(*leaves, lam, None, lengths=[n])
        torch.autograd.grad(o, leaves, do)

    def sp_f():
        with torch.no_grad():
            sp.sp_lightning_attention(*leaves, lam, None, lengths=[n])

    t0 = time.perf_counter()
    r = {k_: round(ev_time(f), 3) for k_, f in (("plain", plain), ("plain_fwd", plain_fwd), ("sp", sp_fb),
                                                 ("sp_fwd", sp_f), ("plain2", plain), ("sp2", sp_fb))}
    print(n, r, f"host {time.perf_counter() - t0:.2f}s", flush=True)
    del q, k, v, do, leaves
    torch.cuda.empty_cache()
