"""Benchmark: Lightning Attention fwd+bwd tokens/s vs sequence length (TNL-1B shape).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the metric's own config): the TNL-1B
attention core -- H=16 heads, d=128, bf16 operands with fp32 accumulation,
per-head decay lam_h = decay_rate(h, l=1, H=16, L=16) -- at a FIXED 64K tokens
per batch for every sequence length n in {1K, 2K, ..., 128K} (batch = 65536/n;
n=128K runs at batch=1, i.e. 131072 tokens).  One STEP = forward + backward at
every sequence length of the sweep, on synthetic standard-normal/sqrt(d)
inputs resident in HBM.  Every per-n working set (268 MB per tensor) exceeds
the 126 MB L2, so no flush is needed between timed iterations.

``value`` = total tokens of the sweep / device time (CUDA events, max over
ranks); the per-n curve is in ``sweep``.  Under torchrun (N > 1) every rank
runs the same per-GPU workload on its own batch x head shard (no collective:
heads and batch are independent), so scaling is weak.

``--impl reference`` times the reference's own CPU algorithm (the oracle's
restatement of kernels.py:253-334, numpy/OpenBLAS, fp32 "working") on the
host cores with one process per core, on a bounded sample of the same
workload, and prints the same line with ``"impl": "reference"``.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "lightning-attn fwd+bwd tokens/s vs seqlen 1K–128K (TNL-1B); % of bf16 peak"
UNIT = "tokens/s"
H, D, L_LAYERS, TOKENS = 16, 128, 16, 65536
SEQ_LENS = (1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072)
FLOPS_PER_HEAD_TOKEN = 28 * D * D          # fwd 8d^2 + bwd 20d^2
BYTES_PER_HEAD_TOKEN = 22 * D              # 11 d-element rows in bf16 (compulsory HBM)
PASS_BYTES_PER_HEAD_TOKEN = 4 * D * 2      # one pass: read 3 rows + write 1 row, bf16


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def lams() -> list[float]:
    from paper_2405_17381_b200.positional import decay_rate

    return [decay_rate(h, 1, H, L_LAYERS) for h in range(1, H + 1)]


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------
# clocks sampled during the timed region
# ----------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(gpu_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
        rows = [r for r in rows if len(r) == 6 and r[0].strip().isdigit()]
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for name, val in zip(names, r[2:]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": int(statistics.median(sm)), "sm_max_mhz": int(rows[0][1]), "reasons": sorted(reasons),
                "samples": len(rows)}


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2405_17381_b200 import ops

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    lam_dev = ops.decay_tensor(lams(), H, device)
    seq_lens = [n for n in args.seq_lens]
    gen = torch.Generator(device=device).manual_seed(1234 + rank)

    def make(n):
        b = max(1, TOKENS // n)
        shape = (b, H, n, D)
        return [(torch.randn(shape, device=device, generator=gen, dtype=torch.float32) / D ** 0.5).to(torch.bfloat16)
                for _ in range(4)]

    # pre-allocate the per-n inputs once (not part of a step); 4 x 268 MB per n
    inputs = {n: make(n) for n in seq_lens}
    tokens = {n: inputs[n][0].shape[0] * n for n in seq_lens}
    stream = torch.cuda.current_stream(device)

    def step(record=None):
        for n in seq_lens:
            q, k, v, do = inputs[n]
            if record is not None:
                record[n][0].record(stream)
            # what the autograd op does: the forward hands its per-segment states to the backward
            _, seg = ops.la_forward(q, k, v, None, lam_dev=lam_dev, want_seg_states=True)
            if record is not None:
                record[n][1].record(stream)
            ops.la_backward(q, k, v, do, None, lam_dev=lam_dev, fwd_seg_states=seg)
            if record is not None:
                record[n][2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    ev = {n: [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)] for n in seq_lens}
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for s in range(args.steps):
        step({n: ev[n][s] for n in seq_lens})
    t1.record(stream)
    torch.cuda.synchronize()
    clock = clocks.stop()
    if world > 1:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([total_ms], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    pk = peaks()
    sweep = {}
    for n in seq_lens:
        fwd = statistics.median(ev[n][s][0].elapsed_time(ev[n][s][1]) for s in range(args.steps))
        bwd = statistics.median(ev[n][s][1].elapsed_time(ev[n][s][2]) for s in range(args.steps))
        tok_s = tokens[n] / ((fwd + bwd) / 1e3)
        sweep[str(n)] = {
            "batch": tokens[n] // n, "fwd_ms": round(fwd, 4), "bwd_ms": round(bwd, 4),
            "tokens_per_s": round(tok_s), "pct_bf16_peak": round(100 * tok_s * H * FLOPS_PER_HEAD_TOKEN
                                                                 / (pk["bf16_tflops"] * 1e12), 2),
            "pct_hbm_roofline": round(100 * tok_s * H * BYTES_PER_HEAD_TOKEN / (pk["hbm_gbs"] * 1e9), 2),
        }
    # per-step device time (first n's fwd start -> last n's bwd end): shows the clock drift inside the
    # timed region once the board reaches its power cap (sw_power_cap)
    step_ms = [round(ev[seq_lens[0]][s][0].elapsed_time(ev[seq_lens[-1]][s][2]), 3) for s in range(args.steps)]
    step_tokens = sum(tokens.values()) * world
    value = step_tokens * args.steps / (total_ms / 1e3)

    # dominant kernel: the pass (one la_fwd = one pass over q,k,v -> o), timed alone on the same stream
    roof = pass_roofline(ops, inputs[args.roofline_n], lam_dev, stream, pk)
    launches = sum(ops.launch_count(tuple(inputs[n][0].shape), which="fwd")
                   + ops.launch_count(tuple(inputs[n][0].shape), which="bwd_saved") for n in seq_lens) * args.steps

    e2e = None if args.no_e2e else run_e2e(ops, seq_lens, tokens, lam_dev, device, min(args.steps, args.e2e_steps),
                                           world)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = cpu_baseline(args.cpu_seconds) if (world == 1 and not args.no_cpu) else None
    del inputs
    torch.cuda.empty_cache()
    rows = None if args.no_rows else measure_rows(ops, device, stream, pk)
    flat = sweep[str(seq_lens[-1])]["tokens_per_s"] / sweep[str(seq_lens[0])]["tokens_per_s"]
    line = {
        "metric": METRIC, "value": round(value), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "TNL-1B attention core (BASELINE configs[2]): H=16, d=128, fixed 64K tokens/batch, "
                               "fwd+bwd at each n of the sweep per step",
                   "heads": H, "head_dim": D, "tokens_per_batch": TOKENS, "seq_lens": seq_lens,
                   "lam": "decay_rate(h, l=1, H=16, L=16)", "parallelism": f"batchxhead-shard x{world}",
                   "l2": "inputs larger than L2 (268 MB per tensor per n)"},
        "pct_bf16_peak": round(100 * value / world * H * FLOPS_PER_HEAD_TOKEN / (pk["bf16_tflops"] * 1e12), 2),
        "flatness_128k_over_1k": round(flat, 3),
        "step_ms": step_ms,
        "sweep": sweep,
        "roofline": roof,
        "gpu_launches": launches,
        "e2e": e2e,
        "clocks": clock,
        "cpu_baseline": cpu,
        "rows": rows,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def _time_ms(fn, stream, reps=10, warm=3) -> float:
    import torch

    for _ in range(warm):
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def measure_rows(ops, device, stream, pk) -> dict:
    """SURVEY.md §8(f) rows at the TNL-1B shape (d_model 2048 = 16 heads x 128), bf16:
    recurrent decode (state traffic vs HBM peak), the GLA layer's element-wise stages (bytes moved
    vs HBM peak), and the whole GLA layer fwd+bwd (cuBLAS projections + these kernels + the core)."""
    import torch

    from paper_2405_17381_b200 import gla
    from paper_2405_17381_b200.positional import decay_rate

    out = {}
    g = torch.Generator(device=device).manual_seed(7)
    rnd = lambda *shape: (torch.randn(*shape, device=device, generator=g) * 0.5).to(torch.bfloat16)  # noqa: E731
    lam = [decay_rate(h, 1, H, L_LAYERS) for h in range(1, H + 1)]
    # decode: 256 sequences x 16 heads, one token each per step; fp32 states (256 MB, > L2) read + written
    # once per step
    bsz = 256
    q, k, v = rnd(bsz, H, D), rnd(bsz, H, D), rnd(bsz, H, D)
    kv = torch.zeros(bsz, H, D, D, device=device, dtype=torch.float32)
    lam_dev = ops.decay_tensor(lam, H, device)
    # a decode step is a few microseconds of GPU work, below the host's per-call overhead: time it as a
    # CUDA graph of 32 steps (what a serving loop replays), per-step time = graph time / 32
    steps_per_graph = 32
    for _ in range(3):
        ops.la_decode(q, k, v, None, kv, lam_dev=lam_dev)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(steps_per_graph):
            ops.la_decode(q, k, v, None, kv, lam_dev=lam_dev)
    ms = _time_ms(graph.replay, stream, reps=10) / steps_per_graph
    state_bytes = bsz * H * D * D * 4 * 2
    out["decode"] = {"batch": bsz, "heads": H, "head_dim": D, "ms_per_step": round(ms, 5), "timing": "CUDA graph of 32 steps",
                     "tokens_per_s": round(bsz / (ms / 1e3)), "state_gbs": round(state_bytes / (ms / 1e3) / 1e9, 1),
                     "frac_hbm": round(state_bytes / (ms / 1e3) / 1e9 / pk["hbm_gbs"], 3)}
    # GLA stages on [8, 8192, 2048] (64K tokens), LRPE on
    b, n, w = 8, 8192, H * D
    row_bytes = b * n * w * 2
    qp, kp, a, u, dgd = (rnd(b, n, w) for _ in range(5))
    theta = torch.tensor([10000.0 ** (-2.0 * j / D) for j in range(D // 2)], dtype=torch.float64, device=device)
    stages = {}
    ms = _time_ms(lambda: ops.gla_prologue(qp, kp, H, theta=theta), stream)
    stages["prologue"] = (ms, 4 * row_bytes)
    gated, raw = ops.gla_epilogue(a, u, H)
    ms = _time_ms(lambda: ops.gla_epilogue(a, u, H), stream)
    stages["epilogue"] = (ms, 3 * row_bytes)
    ms = _time_ms(lambda: ops.gla_epilogue_backward(dgd, a, u, raw, H), stream)
    stages["epilogue_bwd"] = (ms, 5 * row_bytes)
    ms = _time_ms(lambda: ops.gla_prologue_backward(qp, kp, a, u, H, theta=theta), stream)
    stages["prologue_bwd"] = (ms, 6 * row_bytes)
    out["gla_stages"] = {k: {"ms": round(t, 4), "gbs": round(by / (t / 1e3) / 1e9, 1),
                             "frac_hbm": round(by / (t / 1e3) / 1e9 / pk["hbm_gbs"], 3)} for k, (t, by) in stages.items()}
    # BASELINE configs[1]: the TNL-385M attention shape (H = 8, d = 128), n = 2K..16K at 64K tokens/batch
    cfg385 = {}
    lam8 = ops.decay_tensor([decay_rate(h, 1, 8, 24) for h in range(1, 9)], 8, device)
    for n385 in (2048, 4096, 8192, 16384):
        bt = TOKENS // n385
        qq, kk, vv, dd = (rnd(bt, 8, n385, D) for _ in range(4))

        def fb():
            _, seg = ops.la_forward(qq, kk, vv, None, lam_dev=lam8, want_seg_states=True)
            ops.la_backward(qq, kk, vv, dd, None, lam_dev=lam8, fwd_seg_states=seg)

        t = _time_ms(fb, stream, reps=5)
        cfg385[str(n385)] = {"batch": bt, "ms_fwd_bwd": round(t, 4), "tokens_per_s": round(TOKENS / (t / 1e3)),
                          "pct_bf16_peak": round(100 * TOKENS / (t / 1e3) * 8 * FLOPS_PER_HEAD_TOKEN
                                                 / (pk["bf16_tflops"] * 1e12), 2)}
        del qq, kk, vv, dd
    out["tnl385m_attention"] = cfg385
    # BASELINE configs[3] on one GPU (TNL-7B attention shape: 32 heads, d 128, L = 30), fixed 64K tokens;
    # at N GPUs the heads shard 32 / N per rank with no collective, so this is the per-GPU-equivalent line
    cfg7 = {}
    lam32 = ops.decay_tensor([decay_rate(h, 1, 32, 30) for h in range(1, 33)], 32, device)
    for n7 in (2048, 8192, 32768):
        bt = TOKENS // n7
        qq, kk, vv, dd = (rnd(bt, 32, n7, D) for _ in range(4))

        def fb7():
            _, seg = ops.la_forward(qq, kk, vv, None, lam_dev=lam32, want_seg_states=True)
            ops.la_backward(qq, kk, vv, dd, None, lam_dev=lam32, fwd_seg_states=seg)

        t = _time_ms(fb7, stream, reps=5)
        cfg7[str(n7)] = {"batch": bt, "ms_fwd_bwd": round(t, 4), "tokens_per_s": round(TOKENS / (t / 1e3)),
                         "pct_bf16_peak": round(100 * TOKENS / (t / 1e3) * 32 * FLOPS_PER_HEAD_TOKEN
                                                / (pk["bf16_tflops"] * 1e12), 2)}
        del qq, kk, vv, dd
    out["tnl7b_attention_1gpu"] = cfg7
    # BASELINE configs[0] (the reference's CPU-runnable parity case): batch 1, H 4, n 1024, d 64, fp32 on
    # the precision (SIMT) path, lam (1, 0.99, 0.9, 0.5); latency-bound (4 sequences), so no roofline
    c1 = [torch.randn(1, 4, 1024, 64, device=device, generator=g) * 0.5 for _ in range(4)]
    lam1 = ops.decay_tensor([1.0, 0.99, 0.9, 0.5], 4, device)

    def fb1():
        ops.la_forward(*c1[:3], None, lam_dev=lam1)
        ops.la_backward(*c1, None, lam_dev=lam1)

    t1 = _time_ms(fb1, stream)
    out["config1_fp32"] = {"shape": [1, 4, 1024, 64], "ms_fwd_bwd": round(t1, 4),
                           "tokens_per_s": round(1024 / (t1 / 1e3)), "path": "simt fp32 (1e-4 parity path)"}
    # the whole GLA layer, fwd + bwd through autograd
    x = rnd(b, n, w).requires_grad_(True)
    ws = gla.GlaWeights(*(rnd(w, w).mul_(w ** -0.5 * 2).requires_grad_(True) for _ in range(5)))

    def layer():
        y = gla.gla_forward(x, ws, lam, H, theta=theta)
        y.backward(dgd)

    ms = _time_ms(layer, stream, reps=5)
    out["gla_layer"] = {"shape": [b, n, w], "ms_fwd_bwd": round(ms, 3), "tokens_per_s": round(b * n / (ms / 1e3)),
                        "path": "cuBLAS projections + la_gla_* stages + la_fwd/la_bwd core (LRPE on, gate on)"}
    return out


def pass_roofline(ops, tensors, lam_dev, stream, pk) -> dict:
    import torch

    q, k, v, _ = tensors
    reps = 10
    for _ in range(3):
        ops.la_forward(q, k, v, None, lam_dev=lam_dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(stream)
        ops.la_forward(q, k, v, None, lam_dev=lam_dev)
        b.record(stream)
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    head_tokens = q.shape[0] * q.shape[1] * q.shape[2]
    algo = head_tokens * PASS_BYTES_PER_HEAD_TOKEN
    achieved = algo / (ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("pass_dram_bytes_per_launch")
    return {"kernel": "la pass (one la_fwd: q,k,v -> o)", "bound": "hbm", "achieved": round(achieved, 1),
            "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
            "traffic": traffic, "algorithmic_bytes": algo, "launch_ms": round(ms, 4),
            "shape": list(q.shape), "peak_source": pk["source"]}


def run_e2e(ops, seq_lens, tokens, lam_dev, device, steps, world, pieces=4) -> dict:
    """Same metric through the public API with pinned HOST buffers, H2D + D2H inside the timed region.

    Each n's batch is cut into ``pieces`` independent (batch or head) slices, pipelined over three
    streams: H2D of slice i+1 and D2H of slice i-1 overlap the kernels of slice i (PCIe is full
    duplex), so the step is bounded by the link, not by copy + compute + copy in series.
    """
    import torch

    maxel = max(tokens.values()) * H * D
    host_in = [torch.empty(maxel, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
    host_out = [torch.empty(maxel, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
    for t in host_in:
        t.normal_(0, D ** -0.5)
    comp = torch.cuda.current_stream(device)
    h2d_s, d2h_s = torch.cuda.Stream(device), torch.cuda.Stream(device)

    def slices(n):
        b = tokens[n] // n
        views = [h[:tokens[n] * H * D].view(b, H, n, D) for h in host_in + host_out]
        if b > 1:  # batch slices (contiguous in host memory)
            m = min(pieces, b)
            cut = [(i * b // m, (i + 1) * b // m) for i in range(m)]
            return [([v[lo:hi] for v in views], lam_dev) for lo, hi in cut if hi > lo]
        cut = [(i * H // pieces, (i + 1) * H // pieces) for i in range(pieces)]  # batch 1: head slices (contiguous)
        return [([v[:, lo:hi] for v in views], lam_dev[lo:hi]) for lo, hi in cut if hi > lo]

    def one(n):
        moved = 0
        for sl, lam in slices(n):
            hin, hout = sl[:4], sl[4:]
            with torch.cuda.stream(h2d_s):
                dev_in = [h.to(device, non_blocking=True) for h in hin]
                ready = torch.cuda.Event()
                ready.record(h2d_s)
            comp.wait_event(ready)
            o, seg = ops.la_forward(*dev_in[:3], None, lam_dev=lam, want_seg_states=True)
            dq, dk, dv = ops.la_backward(*dev_in, None, lam_dev=lam, fwd_seg_states=seg)
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(done)
                for h, t in zip(hout, (o, dq, dk, dv)):
                    h.copy_(t, non_blocking=True)
            for t in dev_in:
                t.record_stream(comp)
            for t in (o, dq, dk, dv):
                t.record_stream(d2h_s)
            moved += sum(t.numel() * 2 for t in hin)
        return moved, moved

    for n in seq_lens:  # warm the caching allocator's pools of all three streams at every size
        one(n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h2d = d2h = 0
    a.record(comp)
    for _ in range(steps):
        for n in seq_lens:
            i, o = one(n)
            h2d, d2h = h2d + i, d2h + o
    comp.wait_stream(d2h_s)
    b.record(comp)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    value = sum(tokens.values()) * steps * world / (ms / 1e3)
    return {"value": round(value), "unit": UNIT, "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
            "steps": steps, "path": "ops.la_forward/la_backward (C ABI) from pinned host buffers, "
                                    f"{pieces} slices per n pipelined over H2D / compute / D2H streams"}


# ----------------------------------------------------------------------------
# CPU baseline / reference arm: the reference's tiled algorithm on host cores
# ----------------------------------------------------------------------------


def _cpu_unit(args):
    n, d, lam, seed = args
    from threadpoolctl import threadpool_limits

    from oracle import linattn_oracle as orc  # the reference's algorithm, restated (CPU baseline only)

    rng = np.random.default_rng(seed)
    q, k, v, do = (rng.standard_normal((n, d)).astype(np.float32) / np.sqrt(d) for _ in range(4))
    with threadpool_limits(limits=1):  # the reference's own policy (bench.py:36,57)
        t0 = time.perf_counter()
        orc.tiled_forward(q, k, v, lam, d, dtype=np.float32)
        orc.tiled_backward(q, k, v, do, lam, d, dtype=np.float32)
        return time.perf_counter() - t0


class CpuPool:
    """One warmed process per host core, each pinned to one BLAS thread (the reference's policy)."""

    def __init__(self, cores: int):
        from concurrent.futures import ProcessPoolExecutor

        self.cores = cores
        self.ex = ProcessPoolExecutor(max_workers=cores)
        self.lam = lams()

    def run(self, n_units: int, n: int) -> float:
        jobs = [(n, D, self.lam[i % H], i) for i in range(n_units)]
        t0 = time.perf_counter()
        list(self.ex.map(_cpu_unit, jobs, chunksize=1))
        return time.perf_counter() - t0

    def close(self):
        self.ex.shutdown()


CPU_N = 8192


def cpu_baseline(budget_s: float) -> dict:
    """Bounded sample of the workload on the host cores, reported beside the GPU number."""
    cores = len(os.sched_getaffinity(0))
    pool = CpuPool(cores)
    try:
        for _ in range(2):
            first = pool.run(H, CPU_N)  # warm every worker
        units = H * max(1, int((budget_s / 3) / max(first, 1e-3)))
        walls = [pool.run(units, CPU_N) for _ in range(3)]
    finally:
        pool.close()
    wall = statistics.median(walls)
    return {"value": round(units * CPU_N / wall / H, 1), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{units} (batch,head) units of n={CPU_N}, d={D}, fp32 fwd+bwd, median of 3; one process per "
                      "core x 1 BLAS thread; tokens/s = head-tokens/s / H (layer tokens)",
            "wall_s": round(wall, 3)}


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    pool = CpuPool(cores)
    # one step = the sweep's n = 8192 batch (8 sequences x 16 heads = 128 units), handed out one unit at a
    # time so the strongly decaying heads (subnormal-heavy on the CPU) do not leave cores idle
    units = (TOKENS // CPU_N) * H
    try:
        for _ in range(args.warmup):
            pool.run(units, CPU_N)
        walls = [pool.run(units, CPU_N) for _ in range(args.steps)]
    finally:
        pool.close()
    total = sum(walls)
    value = units * CPU_N * len(walls) / total / H
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * total / len(walls), 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": "TNL-1B attention core (BASELINE configs[2]) on host cores: H=16, d=128; step = the "
                               f"sweep's n={CPU_N} batch ({TOKENS // CPU_N} sequences x {H} heads), fwd+bwd, over "
                               f"{cores} processes",
                   "heads": H, "head_dim": D, "seq_len": CPU_N, "batch": TOKENS // CPU_N,
                   "parallelism": f"{cores} processes x 1 BLAS thread"},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{units} (batch, head) units of n={CPU_N} per step; reference tiled algorithm "
                                   "(oracle restatement of kernels.py:253-334), numpy/OpenBLAS fp32"},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--seq-lens", type=lambda s: [int(x) for x in s.split(",")], default=list(SEQ_LENS))
    ap.add_argument("--roofline-n", type=int, default=8192)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-rows", action="store_true", help="skip the decode / GLA-stage / GLA-layer measurements")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.roofline_n not in args.seq_lens:
        args.roofline_n = args.seq_lens[len(args.seq_lens) // 2]
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
