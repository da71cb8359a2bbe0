"""Each kernel family alone, back to back for ~3 s: per-call time over time (CUDA events every 50 calls)
beside nvidia-smi power / clocks / throttle reasons -- which part of the step draws the power that the
board's sustained limit then throttles."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate
dev = torch.device("cuda", 0)
H, D = 16, 128
lam = ops.decay_tensor([decay_rate(h, 1, H, 16) for h in range(1, H + 1)], H, dev)
q, k, v, do = (torch.randn(8, H, 8192, D, device=dev, dtype=torch.bfloat16) for _ in range(4))
arms = {
    "fwd (pass kernel)": lambda: ops.la_forward(q, k, v, None, lam_dev=lam),
    "bwd dq (pass kernel)": lambda: ops.la_backward(q, k, v, do, None, lam_dev=lam, parts="dq"),
    "bwd dkdv (sweep)": lambda: ops.la_backward(q, k, v, do, None, lam_dev=lam, parts="dkdv"),
}
for name, fn in arms.items():
    time.sleep(3.0)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks.mem,clocks_event_reasons.sw_power_cap,"
                            "clocks_event_reasons.hw_slowdown", "--format=csv,noheader", "-lms", "100"],
                           stdout=subprocess.PIPE, text=True)
    t_end = time.time() + 3.0
    times = []
    while time.time() < t_end:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 50)
    smi.terminate()
    out, _ = smi.communicate()
    rows = [r.split(", ") for r in out.strip().splitlines()]
    pw = [float(r[0].split()[0]) for r in rows if r and r[0].split()[0].replace(".", "").isdigit()]
    caps = sum(1 for r in rows if len(r) > 3 and "Active" == r[3].strip())
    print(f"{name}: ms/call first {times[0]:.4f} -> last {times[-1]:.4f} (min {min(times):.4f}, n={len(times)}); "
          f"power max {max(pw):.0f} W median {sorted(pw)[len(pw) // 2]:.0f} W; sm_mhz {rows[len(rows) // 2][1]} "
          f"mem {rows[len(rows) // 2][2]}; power-cap samples {caps}/{len(rows)}", flush=True)
    print("   per-50-call times:", " ".join(f"{t:.3f}" for t in times[:: max(1, len(times) // 16)]), flush=True)
