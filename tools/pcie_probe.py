"""PCIe copy bandwidth from pinned host memory: H2D on 1 vs 2 streams, and H2D + D2H together."""
import time
import torch

dev = torch.device("cuda", 0)
MB = 1 << 20
n = 256 * MB // 2
hs = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
ds = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(4)]
streams = [torch.cuda.Stream() for _ in range(4)]


def run(pairs, reps=5):
    for _ in range(2):
        for fn, s in pairs:
            with torch.cuda.stream(s):
                fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        for fn, s in pairs:
            with torch.cuda.stream(s):
                fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


h2d = lambda i: (lambda: ds[i].copy_(hs[i], non_blocking=True))  # noqa: E731
d2h = lambda i: (lambda: hs[i].copy_(ds[i], non_blocking=True))  # noqa: E731
t = run([(h2d(0), streams[0]), (h2d(1), streams[0])])
print(f"H2D 1 stream : {2 * 256 / 1024 / t:.1f} GB/s")
t = run([(h2d(0), streams[0]), (h2d(1), streams[1])])
print(f"H2D 2 streams: {2 * 256 / 1024 / t:.1f} GB/s")
t = run([(d2h(2), streams[2]), (d2h(3), streams[2])])
print(f"D2H 1 stream : {2 * 256 / 1024 / t:.1f} GB/s")
t = run([(h2d(0), streams[0]), (h2d(1), streams[0]), (d2h(2), streams[2]), (d2h(3), streams[2])])
print(f"H2D+D2H      : {2 * 256 / 1024 / t:.1f} GB/s each way")
t = run([(h2d(0), streams[0]), (h2d(1), streams[1]), (d2h(2), streams[2]), (d2h(3), streams[3])])
print(f"H2D+D2H x2   : {2 * 256 / 1024 / t:.1f} GB/s each way")
