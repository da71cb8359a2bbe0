"""Sequence parallelism: one long sequence split across ranks, exact.

Each rank holds a contiguous slice of the positions of every (batch, head)
sequence.  Lightning attention only couples slices through the d x d carried
state (kernels.py:1-35), so the exchange is tiny and independent
of the slice length:

forward (rank p of P, slice length n_p)
    D_p       = local summary  sum_{s in slice} lam^(end-1-s) k_s v_s^T    (la_fwd_state)
    exchange  KV_in(p) = sum_{q<p} lam^(n_{q+1} + .. + n_{p-1}) D_q         (decayed prefix)
    o_p       = LA(q_p, k_p, v_p; kv_in = KV_in(p))                         (la_fwd_ex, LA_FLAG_RESUME)

backward
    R_p       = local adjoint summary  sum_{t in slice} lam^(t-start+1) q_t do_t^T   (la_bwd_state)
    dq_p      = sweep 1 with the forward's kv_in and segment states  -- on a side stream, overlapping
                the exchange below (it needs nothing from the other ranks)
    exchange  dKV_in(p) = sum_{q>p} lam^(n_{p+1} + .. + n_{q-1}) R_q        (decayed suffix)
    (dk, dv)_p = sweep 2 with dkv_in = dKV_in(p)                            (la_bwd_ex, LA_FLAG_RESUME)

Bytes: a rank's summary pass IS the summary pass of its own segments (the library splits each slice
into segments to fill the GPU, and la_fwd_state leaves their summaries in the workspace), so
``LA_FLAG_RESUME`` skips the second one; the forward hands its segment states to the backward's dq
sweep.  Per rank and step that is the single-GPU traffic plus the last segment's summary (2 rows /
nseg per direction) and the exchange, batch*heads*d*d fp32 per rank (1 MiB for TNL-1B at batch 1).

Exchange (``exchange=``):
  "gather"  one all_gather of every rank's summary, then a fixed-order decayed combine on every rank
            (results independent of arrival order; one latency-bound collective);
  "chain"   the P2P neighbour chain of the north star: rank p receives KV_in(p) from p - 1, sends
            lam^(n_p) KV_in(p) + D_p to p + 1 (the backward runs the chain the other way) -- P - 1
            hops of one d x d message each over NVLink.

The local kernels are pluggable (``LocalKernels``): production uses the CUDA library
(``CudaKernels``); the CPU tests plug in the oracle to exercise this host logic under world-size-2
and -3 ``gloo`` groups.
"""

from __future__ import annotations

from typing import Any, Protocol, Sequence

import torch
import torch.distributed as dist

from .errors import ShapeError

EXCHANGES = ("gather", "chain")


class LocalKernels(Protocol):
    def forward_state(self, k, v, lam) -> tuple[Any, Any]: ...              # (D_p, ctx)
    def forward(self, q, k, v, lam, kv_in, ctx) -> tuple[Any, Any]: ...     # (o_p, forward segment states)
    def backward_state(self, q, do, lam) -> tuple[Any, Any]: ...            # (R_p, ctx)
    def begin_dq(self, q, k, v, do, lam, kv_in, seg) -> Any: ...            # handle (may run asynchronously)
    def backward_dkdv(self, q, k, v, do, lam, dkv_in, ctx) -> tuple[Any, Any]: ...
    def finish_dq(self, handle) -> Any: ...


_SIDE: dict = {}


def _side_stream(device) -> "torch.cuda.Stream":
    """One reusable side stream per device (a fresh stream per call would also defeat the caching
    allocator's per-stream block reuse)."""
    key = torch.device(device).index
    st = _SIDE.get(key)
    if st is None:
        st = _SIDE[key] = torch.cuda.Stream(device)
    return st


class CudaKernels:
    """The B200 library (ops.*) -- the production local kernels."""

    def __init__(self, layout: str = "bhnd", backend: str = "auto"):
        self.layout, self.backend = layout, backend

    def _ws(self, t):
        from . import ops
        return ops.new_workspace(tuple(t.shape), t.dtype, layout=self.layout, backend=self.backend, device=t.device)

    def forward_state(self, k, v, lam):
        from . import ops
        ws = self._ws(k)
        return ops.la_forward_state(k, v, None, lam_dev=lam, layout=self.layout, backend=self.backend,
                                    workspace=ws), ws

    def forward(self, q, k, v, lam, kv_in, ctx):
        from . import ops
        return ops.la_forward(q, k, v, None, lam_dev=lam, kv_in=kv_in, layout=self.layout, backend=self.backend,
                              want_seg_states=True, workspace=ctx, resume=True)

    def backward_state(self, q, do, lam):
        from . import ops
        ws = self._ws(q)
        return ops.la_backward_state(q, do, None, lam_dev=lam, layout=self.layout, backend=self.backend,
                                     workspace=ws), ws

    def begin_dq(self, q, k, v, do, lam, kv_in, seg):
        """Sweep 1 on a side stream: it overlaps the adjoint exchange (NCCL on the caller's stream)."""
        from . import ops
        cur = torch.cuda.current_stream(q.device)
        side = _side_stream(q.device)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            dq, _, _ = ops.la_backward(q, k, v, do, None, lam_dev=lam, kv_in=kv_in, layout=self.layout,
                                       backend=self.backend, fwd_seg_states=seg, parts="dq")
        for t in (q, k, v, do, lam, kv_in, seg):
            if t is not None:
                t.record_stream(side)
        return dq, side

    def backward_dkdv(self, q, k, v, do, lam, dkv_in, ctx):
        from . import ops
        _, dk, dv = ops.la_backward(q, k, v, do, None, lam_dev=lam, dkv_in=dkv_in, layout=self.layout,
                                    backend=self.backend, parts="dkdv", workspace=ctx, resume=True)
        return dk, dv

    def finish_dq(self, handle):
        dq, side = handle
        cur = torch.cuda.current_stream(dq.device)
        cur.wait_stream(side)
        dq.record_stream(cur)
        return dq


def _host_staged(x: torch.Tensor, group) -> bool:
    """gloo moves host tensors: a CUDA state crosses it through a host copy (NCCL takes device tensors)."""
    return x.is_cuda and dist.get_backend(group) == "gloo"


def _gather(x: torch.Tensor, group) -> list[torch.Tensor]:
    world = dist.get_world_size(group)
    if _host_staged(x, group):
        h = x.detach().cpu()
        out = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(out, h, group=group)
        return [o.to(x.device) for o in out]
    out = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(out, x.contiguous(), group=group)
    return out


def _decay(lam: torch.Tensor, length: int) -> torch.Tensor:
    """lam^length per head, broadcastable against [batch, heads, d, d]."""
    return torch.pow(lam.to(torch.float64), float(length)).view(1, -1, 1, 1)


def prefix_states(deltas: Sequence[torch.Tensor], lengths: Sequence[int], lam: torch.Tensor, rank: int):
    """KV_in(rank) = sum_{q<rank} lam^(n_{q+1}+..+n_{rank-1}) D_q, combined in rank order."""
    s = torch.zeros_like(deltas[0], dtype=torch.float64)
    for q in range(rank):
        s = _decay(lam, lengths[q]).to(s.device) * s + deltas[q].to(torch.float64)
    return s.to(deltas[0].dtype)


def suffix_states(deltas: Sequence[torch.Tensor], lengths: Sequence[int], lam: torch.Tensor, rank: int):
    """dKV_in(rank) = sum_{q>rank} lam^(n_{rank+1}+..+n_{q-1}) R_q, combined in rank order."""
    s = torch.zeros_like(deltas[0], dtype=torch.float64)
    for q in range(len(deltas) - 1, rank, -1):
        s = _decay(lam, lengths[q]).to(s.device) * s + deltas[q].to(torch.float64)
    return s.to(deltas[0].dtype)


def _chain(delta: torch.Tensor, lengths: Sequence[int], lam: torch.Tensor, group, reverse: bool) -> torch.Tensor:
    """The neighbour chain: receive the entering state from the previous rank (the next one when
    `reverse`), pass lam^(n_p) * entering + delta on.  Returns this rank's entering state."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    src = rank + 1 if reverse else rank - 1
    dst = rank - 1 if reverse else rank + 1
    staged = _host_staged(delta, group)
    entering = torch.zeros_like(delta)
    if 0 <= src < world:
        if staged:
            h = torch.empty_like(delta, device="cpu")
            dist.recv(h, group_src=src, group=group)
            entering = h.to(delta.device)
        else:
            dist.recv(entering, group_src=src, group=group)
    if 0 <= dst < world:
        out = (_decay(lam, lengths[rank]).to(delta.device) * entering.to(torch.float64)
               + delta.to(torch.float64)).to(delta.dtype)
        dist.send(out.cpu() if staged else out.contiguous(), group_dst=dst, group=group)
    return entering


def _exchange(delta, lengths, lam, group, exchange: str, reverse: bool):
    if group is None:  # one rank, no process group: nothing enters from outside the slice
        return torch.zeros_like(delta)
    rank = dist.get_rank(group)
    if exchange == "chain":
        return _chain(delta, lengths, lam, group, reverse)
    gathered = _gather(delta, group)
    return suffix_states(gathered, lengths, lam, rank) if reverse else prefix_states(gathered, lengths, lam, rank)


def _lengths(n_local: int, group) -> list[int]:
    if group is None:
        return [n_local]
    world = dist.get_world_size(group)
    t = torch.tensor([n_local], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


class SequenceParallelLightning(torch.autograd.Function):
    """o_p = slice p of LA(q, k, v) for the full sequence; inputs are this rank's slice."""

    @staticmethod
    def forward(ctx, q, k, v, lam, group, kernels, n_axis, lengths, exchange):
        rank = dist.get_rank(group) if group is not None else 0
        world = dist.get_world_size(group) if group is not None else 1
        if lengths is None:
            lengths = _lengths(q.shape[n_axis], group)
        elif len(lengths) != world or lengths[rank] != q.shape[n_axis]:
            raise ShapeError(f"lengths {list(lengths)} do not match this group / this rank's slice "
                             f"({q.shape[n_axis]} positions on rank {rank})")
        delta, fctx = kernels.forward_state(k, v, lam)
        kv_in = _exchange(delta, lengths, lam, group, exchange, reverse=False)
        o, seg = kernels.forward(q, k, v, lam, kv_in, fctx)
        ctx.save_for_backward(q, k, v, lam, kv_in, seg)
        ctx.group, ctx.kernels, ctx.lengths, ctx.exchange = group, kernels, lengths, exchange
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, lam, kv_in, seg = ctx.saved_tensors
        kernels = ctx.kernels
        do = do.contiguous().to(q.dtype)
        r, bctx = kernels.backward_state(q, do, lam)
        handle = kernels.begin_dq(q, k, v, do, lam, kv_in, seg)
        dkv_in = _exchange(r, ctx.lengths, lam, ctx.group, ctx.exchange, reverse=True)
        dk, dv = kernels.backward_dkdv(q, k, v, do, lam, dkv_in, bctx)
        dq = kernels.finish_dq(handle)
        return dq, dk, dv, None, None, None, None, None, None


def sp_lightning_attention(q, k, v, lam, group=None, *, layout: str = "bhnd", kernels: LocalKernels | None = None,
                           lengths: Sequence[int] | None = None, exchange: str = "gather"):
    """Sequence-parallel lightning attention over ``group`` (default: WORLD when a process group is
    initialised, else a single rank).

    ``q, k, v``: this rank's contiguous slice of positions, [b, h, n_p, d] ("bhnd") or [b, n_p, h, d]
    ("bnhd"); ranks hold slices in rank order.  ``lam``: one decay per head -- anything
    ``ops.decay_tensor`` accepts; a tensor is used as is only when it already is a contiguous float64
    tensor of one value per head on the inputs' device.  ``lengths``: every rank's slice length in rank
    order, when the caller knows them (fixed slicing); otherwise they are exchanged with one small
    all_gather per call, whose read-back synchronises the host with the stream.  ``exchange``: "gather"
    or "chain" (see the module docstring).
    """
    if layout not in ("bhnd", "bnhd"):
        raise ShapeError(f"layout must be 'bhnd' or 'bnhd', got {layout!r}")
    if exchange not in EXCHANGES:
        raise ShapeError(f"exchange must be one of {EXCHANGES}, got {exchange!r}")
    if group is None and dist.is_available() and dist.is_initialized():
        group = dist.group.WORLD
    heads = q.shape[1] if layout == "bhnd" else q.shape[2]
    if not (isinstance(lam, torch.Tensor) and lam.dtype == torch.float64 and lam.device == q.device
            and lam.numel() == heads and lam.is_contiguous()):
        from .ops import decay_tensor
        lam = decay_tensor(lam, heads, q.device)
    if kernels is None:
        kernels = CudaKernels(layout=layout)
    return SequenceParallelLightning.apply(q, k, v, lam, group, kernels, 2 if layout == "bhnd" else 1,
                                           None if lengths is None else [int(x) for x in lengths], exchange)
