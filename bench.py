"""Benchmark: Lightning Attention fwd+bwd tokens/s vs sequence length (TNL-1B shape).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--gpus N`` (N > 1) without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks on this node (127.0.0.1 rendezvous) and fails loudly
when fewer than N CUDA devices are visible; under torchrun WORLD_SIZE must equal N.

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

Beside the headline line's sweep, ``multi`` carries the two multi-GPU configurations, run by every
rank and timed as the max over ranks:
  * ``tnl7b_heads`` (BASELINE configs[3]): TNL-7B attention, 32 heads sharded 32 / N per rank, no
    collective, 64K tokens per batch at n = 2K / 8K / 32K -- strong scaling (fixed layer work);
  * ``sequence_parallel`` (configs[4]): TNL-1B attention at 512K and 1M tokens (batch 1), each
    sequence split over the N ranks through ``sp.sp_lightning_attention`` (all_gather exchange of the
    d x d summaries, NCCL) -- strong scaling; plus the same sequence on one GPU for the efficiency.

``--impl reference`` times the reference's own CPU implementation -- the stock
``linattn.kernels.lightning_forward_decay`` / ``lightning_backward_decay``
(kernels.py:253-334, precision "working" = fp32, its _prep and ensure_finite
included) installed unmodified in ``baseline/_ref`` -- on the host cores with one
process per core (threadpool_limits(1), the reference's own policy, bench.py:36,57),
each step one sequence at every n of the sweep x all 16 heads, and prints the
same line with ``"impl": "reference"``.  Without ``baseline/_ref`` it falls back
to the oracle's restatement of the same algorithm (kind "port").
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


def head_shard(rank: int, world: int, heads: int) -> tuple[int, int]:
    """Contiguous head range [lo, hi) of `rank` (batch x head sharding, no collective: SPEC.md:256)."""
    return rank * heads // world, (rank + 1) * heads // world


def sp_slice(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous position range [lo, hi) of `rank` in sequence-parallel mode, 128-row (chunk) aligned."""
    chunks = (n_total + 127) // 128
    lo, hi = rank * chunks // world, (rank + 1) * chunks // world
    return min(n_total, lo * 128), min(n_total, hi * 128)


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_relaunch(args) -> None:
    """``--gpus N`` outside torchrun: re-exec under torch.distributed.run with N ranks on this node."""
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={os.environ['WORLD_SIZE']}")
        return
    if args.gpus <= 1 or args.impl == "reference":  # the reference arm is host-only: rank 0's work, no ranks
        return
    if os.environ.get("LA_BENCH_LAUNCH_PROBE") != "1" and os.environ.get("LA_BENCH_SHARED_GPU") != "1":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def launch_probe(args) -> None:
    """LA_BENCH_LAUNCH_PROBE=1 (CPU tests): the multi-rank plumbing without GPU work -- rendezvous, the
    shard plans of every rank, and the max-over-ranks reduction -- printed by rank 0 as one JSON line."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    mine = torch.tensor([float(rank + 1)], dtype=torch.float64)  # a rank-dependent "time"
    plan = torch.tensor([*head_shard(rank, world, 32), *sp_slice(1 << 20, rank, world)], dtype=torch.int64)
    plans = [torch.zeros_like(plan) for _ in range(world)]
    if world > 1:
        dist.all_reduce(mine, op=dist.ReduceOp.MAX)
        dist.all_gather(plans, plan)
    else:
        plans = [plan]
    if rank == 0:
        print(json.dumps({"probe": True, "world": world, "gpus": args.gpus, "max_over_ranks": float(mine.item()),
                          "tnl7b_heads": [p[:2].tolist() for p in plans], "sp_slices": [p[2:].tolist() for p in plans]}))
    if world > 1:
        dist.destroy_process_group()


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
    # LA_BENCH_SHARED_GPU=1 (tests only: tests/test_gpu_bench_ranks.py): every rank on cuda:0 over gloo, to run
    # the multi-rank code path on a one-GPU box -- its numbers are meaningless (the ranks share one GPU)
    shared = os.environ.get("LA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
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

    def reduce_max(ms: float) -> float:  # max over ranks (a host tensor over gloo, a device one over NCCL)
        if world == 1:
            return ms
        t = torch.tensor([ms], device="cpu" if shared else device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_ms = reduce_max(total_ms)

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

    # dominant kernel: the pass (one la_fwd = one pass over q,k,v -> o).  `achieved` uses its launches
    # INSIDE the timed region (the forward events at roofline_n: one la_fwd there is one pass-kernel launch
    # when the sequence is not split), `achieved_alone` the same launch timed alone right after it
    rn = args.roofline_n
    in_region_ms = statistics.mean(ev[rn][s][0].elapsed_time(ev[rn][s][1]) for s in range(args.steps))
    roof = pass_roofline(ops, inputs[rn], lam_dev, stream, pk, in_region_ms)
    launches = sum(ops.launch_count(tuple(inputs[n][0].shape), which="fwd")
                   + ops.launch_count(tuple(inputs[n][0].shape), which="bwd_saved") for n in seq_lens) * args.steps

    e2e = None if args.no_e2e else run_e2e(ops, seq_lens, tokens, lam_dev, device, min(args.steps, args.e2e_steps),
                                           world, reduce_max)
    del inputs
    torch.cuda.empty_cache()
    multi = None if args.no_multi else run_multi(ops, device, world, rank, stream, pk, reduce_max,
                                                 max(1, min(args.steps, args.multi_steps)))
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = cpu_baseline() if (world == 1 and not args.no_cpu) else None
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
        "multi": multi,
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
    # the GLA core forward (§8(f) rank 1): fused (act + LRPE in the pass kernel, q / k written for the backward;
    # and without them, as a prefill needs) vs the two-step path it replaces (la_gla_prologue + la_fwd)
    vv = rnd(b, n, w)

    def two_step():
        q2, k2 = ops.gla_prologue(qp, kp, H, theta=theta)
        ops.la_forward(*(t.view(b, n, H, D) for t in (q2, k2, vv)), None, lam_dev=lam_dev, layout="bnhd")

    t_two = _time_ms(two_step, stream)
    t_fused = _time_ms(lambda: ops.gla_core_forward(qp, kp, vv, None, H, theta=theta, lam_dev=lam_dev), stream)
    t_fused_nq = _time_ms(lambda: ops.gla_core_forward(qp, kp, vv, None, H, theta=theta, lam_dev=lam_dev,
                                                       want_qk=False), stream)
    out["gla_core_fwd"] = {
        "shape": [b, n, w], "lrpe": True, "act": "swish",
        "two_step_ms": round(t_two, 4), "fused_ms": round(t_fused, 4), "fused_no_qk_ms": round(t_fused_nq, 4),
        "speedup": round(t_two / t_fused, 3), "speedup_no_qk": round(t_two / t_fused_nq, 3),
        "rows_moved": {"two_step": 8, "fused": 6, "fused_no_qk": 4},
        "fused_frac_hbm": round(6 * row_bytes / (t_fused / 1e3) / 1e9 / pk["hbm_gbs"], 3)}
    del vv
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
    # the headline sweep's shape with LONG-memory decays (layer 15 of 16: lam_h = exp(-h/32), 0.97 .. 0.61):
    # the summary pass can skip nothing for the slow heads (la_summary.cu), so this is the general-case curve
    lam_long = ops.decay_tensor([decay_rate(h, 15, H, L_LAYERS) for h in range(1, H + 1)], H, device)
    long_rows = {}
    for nl in (1024, 8192, 32768, 131072):
        bt = max(1, TOKENS // nl)
        qq, kk, vv, dd = (rnd(bt, H, nl, D) for _ in range(4))

        def fbl():
            _, seg = ops.la_forward(qq, kk, vv, None, lam_dev=lam_long, want_seg_states=True)
            ops.la_backward(qq, kk, vv, dd, None, lam_dev=lam_long, fwd_seg_states=seg)

        t = _time_ms(fbl, stream, reps=5)
        long_rows[str(nl)] = {"batch": bt, "ms_fwd_bwd": round(t, 4), "tokens_per_s": round(bt * nl / (t / 1e3)),
                              "pct_bf16_peak": round(100 * bt * nl / (t / 1e3) * H * FLOPS_PER_HEAD_TOKEN
                                                     / (pk["bf16_tflops"] * 1e12), 2)}
        del qq, kk, vv, dd
    out["tnl1b_long_memory_decays"] = {"lam": "decay_rate(h, 15, 16, 16)", "rows": long_rows}
    # fp32 ("working" precision, the 1e-4 parity path) at the TNL-1B shape, n = 8K: the tensor-core split pass
    # (la_tc32.cu, the default for fp32 at d = 128) and the SIMT FFMA pass beside it
    q32, k32, v32, d32 = (torch.randn(8, H, 8192, D, device=device, generator=g) / D ** 0.5 for _ in range(4))
    fp32_rows = {}
    for be, path in (("tcgen05", "tcgen05 fp32 (3-term bf16 split, 1e-4 parity path)"),
                     ("simt", "simt fp32 (FFMA)")):
        def fb32():
            _, seg = ops.la_forward(q32, k32, v32, None, lam_dev=lam_dev, want_seg_states=True, backend=be)
            ops.la_backward(q32, k32, v32, d32, None, lam_dev=lam_dev, fwd_seg_states=seg, backend=be)

        t32 = _time_ms(fb32, stream, reps=3 if be == "simt" else 10, warm=1 if be == "simt" else 3)
        fp32_rows[be] = {"ms_fwd_bwd": round(t32, 3), "tokens_per_s": round(8 * 8192 / (t32 / 1e3)), "path": path}
    out["fp32_tnl1b_8k"] = {"shape": [8, H, 8192, D], **fp32_rows}
    del q32, k32, v32, d32
    # BASELINE configs[0] (the reference's CPU-runnable parity case): batch 1, H 4, n 1024, d 64, fp32,
    # lam (1, 0.99, 0.9, 0.5); the default route is the tensor-core split pass on zero-padded d = 128
    # tiles, the SIMT pass timed beside it; latency-bound (4 sequences), so no roofline
    c1 = [torch.randn(1, 4, 1024, 64, device=device, generator=g) * 0.5 for _ in range(4)]
    lam1 = ops.decay_tensor([1.0, 0.99, 0.9, 0.5], 4, device)
    c1_rows = {}
    for be, path in (("tcgen05", "tcgen05 fp32 (3-term bf16 split, default route)"),
                     ("simt", "simt fp32 (FFMA)")):
        def fb1(be=be):
            ops.la_forward(*c1[:3], None, lam_dev=lam1, backend=be)
            ops.la_backward(*c1, None, lam_dev=lam1, backend=be)

        t1 = _time_ms(fb1, stream)
        c1_rows[be] = {"ms_fwd_bwd": round(t1, 4), "tokens_per_s": round(1024 / (t1 / 1e3)), "path": path}
    out["config1_fp32"] = {"shape": [1, 4, 1024, 64], **c1_rows}
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


def pass_roofline(ops, tensors, lam_dev, stream, pk, in_region_ms=None) -> dict:
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
    alone_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    # one launch per la_fwd only when the plan does not split the sequence (summaries + scan otherwise)
    single = ops.launch_count(tuple(q.shape), which="fwd") == 1
    in_region = in_region_ms is not None and single
    ms = in_region_ms if in_region else alone_ms
    head_tokens = q.shape[0] * q.shape[1] * q.shape[2]
    algo = head_tokens * PASS_BYTES_PER_HEAD_TOKEN
    achieved = algo / (ms / 1e3) / 1e9
    achieved_alone = algo / (alone_ms / 1e3) / 1e9
    # DRAM bytes of this launch are not measurable in-process (no CUPTI here): they come from the ncu
    # --set full capture of the same launch committed under profiles/, named in traffic_source
    traffic, source = None, None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        tj = json.loads(prof.read_text())
        traffic = tj.get("pass_dram_bytes_per_launch")
        source = tj.get("source", "profiles/traffic.json")
    return {"kernel": "la pass (one la_fwd: q,k,v -> o)", "bound": "hbm", "achieved": round(achieved, 1),
            "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
            "traffic": traffic, "traffic_source": source, "algorithmic_bytes": algo, "launch_ms": round(ms, 4),
            "timing": "mean launch inside the timed region" if in_region else "timed alone after the region",
            "achieved_alone": round(achieved_alone, 1), "launch_ms_alone": round(alone_ms, 4),
            "frac_alone": round(achieved_alone / pk["hbm_gbs"], 4),
            "shape": list(q.shape), "peak_source": pk["source"]}


def run_e2e(ops, seq_lens, tokens, lam_dev, device, steps, world, reduce_max, pieces=4) -> dict:
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
    ms = reduce_max(a.elapsed_time(b))
    value = sum(tokens.values()) * steps * world / (ms / 1e3)
    return {"value": round(value), "unit": UNIT, "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
            "steps": steps, "path": "ops.la_forward/la_backward (C ABI) from pinned host buffers, "
                                    f"{pieces} slices per n pipelined over H2D / compute / D2H streams"}


def run_multi(ops, device, world, rank, stream, pk, reduce_max, steps) -> dict:
    """BASELINE configs[3] (TNL-7B heads sharded over the ranks) and configs[4] (TNL-1B sequence parallel at
    512K / 1M tokens) -- every rank runs its share; device time (CUDA events) as the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2405_17381_b200 import sp
    from paper_2405_17381_b200.positional import decay_rate

    g = torch.Generator(device=device).manual_seed(4321 + rank)
    rnd = lambda *shape: (torch.randn(*shape, device=device, generator=g) / D ** 0.5).to(torch.bfloat16)  # noqa: E731

    def timed(fn) -> float:
        for _ in range(3):  # warm-up: also lets the caching allocator settle on this row's block sizes
            fn()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return reduce_max(a.elapsed_time(b) / steps)

    out = {}
    # configs[3]: TNL-7B attention (H = 32, d = 128, L = 30), heads sharded 32 / N, 64K tokens per batch
    h7 = 32
    lo, hi = head_shard(rank, world, h7)
    lam7 = ops.decay_tensor([decay_rate(h, 1, h7, 30) for h in range(lo + 1, hi + 1)], hi - lo, device)
    rows7 = {}
    for n in (2048, 8192, 32768):
        b = TOKENS // n
        q, k, v, do = (rnd(b, hi - lo, n, D) for _ in range(4))

        def fb():
            _, seg = ops.la_forward(q, k, v, None, lam_dev=lam7, want_seg_states=True)
            ops.la_backward(q, k, v, do, None, lam_dev=lam7, fwd_seg_states=seg)

        ms = timed(fb)
        tok = TOKENS / (ms / 1e3)
        rows7[str(n)] = {"batch": b, "heads_per_rank": hi - lo, "ms_fwd_bwd": round(ms, 4), "tokens_per_s": round(tok),
                         "tokens_per_s_per_gpu": round(tok / world),
                         "pct_bf16_peak": round(100 * tok * h7 * FLOPS_PER_HEAD_TOKEN
                                                / (world * pk["bf16_tflops"] * 1e12), 2)}
        del q, k, v, do
    out["tnl7b_heads"] = {"workload": "BASELINE configs[3]: TNL-7B attention, H=32, d=128, bf16, fwd+bwd, 64K tokens "
                                      "per batch, heads sharded over the ranks (no collective); strong scaling",
                          "n_gpus": world, "rows": rows7}
    # configs[4]: TNL-1B attention, one sequence of 512K / 1M tokens split over the ranks
    lam_sp = ops.decay_tensor(lams(), H, device)
    group = dist.group.WORLD if world > 1 else None
    rows_sp = {}
    torch.cuda.empty_cache()
    for n_total in (524288, 1048576):
        plo, phi = sp_slice(n_total, rank, world)
        lengths = [sp_slice(n_total, r, world)[1] - sp_slice(n_total, r, world)[0] for r in range(world)]
        q, k, v, do = (rnd(1, H, phi - plo, D) for _ in range(4))
        leaves = [t.requires_grad_(True) for t in (q, k, v)]

        def fb_sp():
            o = sp.sp_lightning_attention(*leaves, lam_sp, group, lengths=lengths)
            torch.autograd.grad(o, leaves, do)

        ms = timed(fb_sp)
        row = {"n_per_rank": phi - plo, "ms_fwd_bwd": round(ms, 4), "tokens_per_s": round(n_total / (ms / 1e3)),
               "pct_bf16_peak": round(100 * n_total / (ms / 1e3) * H * FLOPS_PER_HEAD_TOKEN
                                      / (world * pk["bf16_tflops"] * 1e12), 2)}
        del q, k, v, do, leaves
        torch.cuda.empty_cache()
        # the same sequence on one GPU (rank 0), through the plain entry points: the efficiency baseline
        if rank == 0:
            q1, k1, v1, d1 = (rnd(1, H, n_total, D) for _ in range(4))

            def fb_one():
                _, seg = ops.la_forward(q1, k1, v1, None, lam_dev=lam_sp, want_seg_states=True)
                ops.la_backward(q1, k1, v1, d1, None, lam_dev=lam_sp, fwd_seg_states=seg)

            for _ in range(3):
                fb_one()
                torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(steps):
                fb_one()
            b.record(stream)
            torch.cuda.synchronize()
            one = a.elapsed_time(b) / steps
            row["single_gpu_ms"] = round(one, 4)
            row["single_gpu_tokens_per_s"] = round(n_total / (one / 1e3))
            row["parallel_efficiency"] = round(one / (world * ms), 3)
            del q1, k1, v1, d1
            torch.cuda.empty_cache()
        if world > 1:
            dist.barrier()
        rows_sp[str(n_total)] = row
    out["sequence_parallel"] = {"workload": "BASELINE configs[4]: TNL-1B attention (H=16, d=128, bf16), batch 1, "
                                            "fwd+bwd, the sequence split over the ranks (sp.sp_lightning_attention, "
                                            "all_gather of the d x d summaries over NCCL); strong scaling",
                                "n_gpus": world, "exchange": "gather", "rows": rows_sp}
    return out


# ----------------------------------------------------------------------------
# CPU baseline / reference arm: the reference's own implementation on host cores
# ----------------------------------------------------------------------------

REF_DIR = ROOT / "baseline" / "_ref"


def _ref_init():
    if (REF_DIR / "linattn").is_dir() and str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))


def _ref_kind() -> str:
    return "reference" if (REF_DIR / "linattn" / "kernels.py").exists() else "port"


def _cpu_unit(args):
    """One (sequence, head) unit, fwd + bwd in fp32 ("working"), timed; inputs made outside the timing."""
    n, d, lam, seed = args
    from threadpoolctl import threadpool_limits

    rng = np.random.default_rng(seed)
    q, k, v, do = (rng.standard_normal((n, d)).astype(np.float32) / np.float32(np.sqrt(d)) for _ in range(4))
    with threadpool_limits(limits=1):  # the reference's own policy (bench.py:36,57)
        if _ref_kind() == "reference":
            # the stock reference, unmodified (baseline/_ref/linattn): its _prep, ensure_finite, tiled sweeps
            from linattn.kernels import AttentionConfig, lightning_backward_decay, lightning_forward_decay

            cfg = AttentionConfig(n=n, d=d, B=None, lam=lam, precision="working")
            t0 = time.perf_counter()
            lightning_forward_decay(q, k, v, cfg)
            lightning_backward_decay(q, k, v, do, cfg)
            return time.perf_counter() - t0
        from oracle import linattn_oracle as orc  # restatement of the same algorithm (CPU baseline only)

        t0 = time.perf_counter()
        orc.tiled_forward(q, k, v, lam, d, dtype=np.float32)
        orc.tiled_backward(q, k, v, do, lam, d, dtype=np.float32)
        return time.perf_counter() - t0


class CpuPool:
    """One warmed process per host core, each pinned to one BLAS thread (the reference's policy)."""

    def __init__(self, cores: int):
        from concurrent.futures import ProcessPoolExecutor

        self.cores = cores
        self.ex = ProcessPoolExecutor(max_workers=cores, initializer=_ref_init)
        self.lam = lams()

    def run_sweep(self, heads) -> float:
        """One sequence at every n of the sweep x the given heads; the longest units first."""
        jobs = sorted(((n, D, self.lam[h], 1000 * h + i) for i, n in enumerate(SEQ_LENS) for h in heads),
                      key=lambda j: -j[0])
        t0 = time.perf_counter()
        list(self.ex.map(_cpu_unit, jobs, chunksize=1))
        return time.perf_counter() - t0

    def close(self):
        self.ex.shutdown()


SWEEP_TOKENS = sum(SEQ_LENS)  # one sequence at every n: 261,120 layer tokens


def _sample_heads(pool, budget_s: float):
    """All 16 heads per n unless one sweep would exceed `budget_s` on these cores; then every other head
    (the decays still span 0.63 .. 5.5e-4).  Returns (heads, warm-up wall)."""
    heads = list(range(H))
    wall = pool.run_sweep(heads)
    if wall > budget_s:
        heads = list(range(0, H, 2))
    return heads, wall


def cpu_baseline() -> dict:
    """Bounded sample of the workload on the host cores, reported beside the GPU number."""
    cores = len(os.sched_getaffinity(0))
    _ref_init()
    pool = CpuPool(cores)
    try:
        heads, _ = _sample_heads(pool, 12.0)
        wall = pool.run_sweep(heads)
    finally:
        pool.close()
    value = SWEEP_TOKENS * len(heads) / H / wall
    return {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": _ref_kind(),
            "sample": f"one sequence at every n of the sweep (1K..128K) x {len(heads)} of the {H} heads, fwd+bwd, "
                      "fp32 'working' precision, one timed sweep after a warm one; one process per core x 1 BLAS "
                      f"thread; tokens/s = layer tokens (head-tokens / {H})",
            "impl": "baseline/_ref linattn.kernels (stock)" if _ref_kind() == "reference" else "oracle port",
            "wall_s": round(wall, 3)}


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    _ref_init()
    pool = CpuPool(cores)
    try:
        heads, _ = _sample_heads(pool, 9.0)  # keeps --steps 20 --warmup 5 within a few minutes
        for _ in range(max(0, args.warmup - 1)):
            pool.run_sweep(heads)
        walls = [pool.run_sweep(heads) for _ in range(args.steps)]
    finally:
        pool.close()
    total = sum(walls)
    value = SWEEP_TOKENS * len(heads) / H * len(walls) / total
    sample = (f"per step: one sequence at every n of the sweep (1K..128K) x {len(heads)} of the {H} heads (TNL-1B "
              f"decays), fwd+bwd, fp32 'working'; {cores} processes x 1 BLAS thread")
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * total / len(walls), 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": "TNL-1B attention core (BASELINE configs[2]) on host cores: H=16, d=128, "
                               "lam=decay_rate(h, 1, 16, 16), fwd+bwd at every n of the 1K..128K sweep (batch 1 per n)",
                   "heads": H, "heads_sampled": len(heads), "head_dim": D, "seq_lens": list(SEQ_LENS),
                   "parallelism": f"{cores} processes x 1 BLAS thread"},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": _ref_kind(), "sample": sample},
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
    ap.add_argument("--multi-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-multi", action="store_true", help="skip the TNL-7B head-shard and sequence-parallel rows")
    ap.add_argument("--no-rows", action="store_true", help="skip the decode / GLA-stage / GLA-layer measurements")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.roofline_n not in args.seq_lens:
        args.roofline_n = args.seq_lens[len(args.seq_lens) // 2]
    maybe_relaunch(args)
    if os.environ.get("LA_BENCH_LAUNCH_PROBE") == "1":
        launch_probe(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
