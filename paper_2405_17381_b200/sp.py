"""Sequence parallelism: one long sequence split across ranks, exact.

Each rank holds a contiguous slice of the positions of every (batch, head)
sequence.  Lightning attention only couples slices through the d x d carried
state (kernels.py:1-35), so the exchange is tiny and independent
of the slice length:

forward (rank p of P, slice length n_p)
    D_p       = local summary  sum_{s in slice} lam^(end-1-s) k_s v_s^T    (la_fwd_state)
    all_gather(D_0 .. D_{P-1})                                              (one NCCL collective)
    KV_in(p)  = sum_{q<p} lam^(n_{q+1} + .. + n_{p-1}) D_q                  (decayed prefix, fixed order)
    o_p       = LA(q_p, k_p, v_p; kv_in = KV_in(p))                         (la_fwd)

backward
    R_p       = local adjoint summary  sum_{t in slice} lam^(t-start+1) q_t do_t^T   (la_bwd_state)
    all_gather(R_0 .. R_{P-1})
    dKV_in(p) = sum_{q>p} lam^(n_{p+1} + .. + n_{q-1}) R_q                  (decayed suffix)
    (dq, dk, dv)_p = LA'(...; kv_in = KV_in(p), dkv_in = dKV_in(p))         (la_bwd)

Messages are batch*heads*d*d fp32 per rank (1 MiB for TNL-1B at batch 1);
the combine order is fixed, so results do not depend on arrival order.  The
gather is a single collective rather than a P-1 hop chain: latency-bound
either way on NVLink/NVSwitch, and the gather keeps every rank symmetric.

The local kernels are pluggable (``LocalKernels``): production uses the CUDA
library (``CudaKernels``); the CPU tests plug in the oracle to exercise this
host logic under a world-size-2 ``gloo`` group.
"""

from __future__ import annotations

from typing import Protocol, Sequence

import torch
import torch.distributed as dist

from .errors import ShapeError


class LocalKernels(Protocol):
    def forward_state(self, k, v, lam): ...
    def backward_state(self, q, do, lam): ...
    def forward(self, q, k, v, lam, kv_in): ...
    def backward(self, q, k, v, do, lam, kv_in, dkv_in): ...


class CudaKernels:
    """The B200 library (ops.*) -- the production local kernels."""

    def __init__(self, layout: str = "bhnd", backend: str = "auto"):
        self.layout, self.backend = layout, backend

    def forward_state(self, k, v, lam):
        from . import ops
        return ops.la_forward_state(k, v, None, lam_dev=lam, layout=self.layout, backend=self.backend)

    def backward_state(self, q, do, lam):
        from . import ops
        return ops.la_backward_state(q, do, None, lam_dev=lam, layout=self.layout, backend=self.backend)

    def forward(self, q, k, v, lam, kv_in):
        from . import ops
        return ops.la_forward(q, k, v, None, lam_dev=lam, kv_in=kv_in, layout=self.layout, backend=self.backend)

    def backward(self, q, k, v, do, lam, kv_in, dkv_in):
        from . import ops
        return ops.la_backward(q, k, v, do, None, lam_dev=lam, kv_in=kv_in, dkv_in=dkv_in, layout=self.layout,
                               backend=self.backend)


def _gather(x: torch.Tensor, group) -> list[torch.Tensor]:
    world = dist.get_world_size(group)
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


def _lengths(n_local: int, group) -> list[int]:
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
    def forward(ctx, q, k, v, lam, group, kernels, n_axis, lengths=None):
        rank = dist.get_rank(group)
        if lengths is None:
            lengths = _lengths(q.shape[n_axis], group)
        elif len(lengths) != dist.get_world_size(group) or lengths[rank] != q.shape[n_axis]:
            raise ShapeError(f"lengths {list(lengths)} do not match this group / this rank's slice "
                             f"({q.shape[n_axis]} positions on rank {rank})")
        delta = kernels.forward_state(k, v, lam)
        kv_in = prefix_states(_gather(delta, group), lengths, lam, rank)
        o = kernels.forward(q, k, v, lam, kv_in)
        ctx.save_for_backward(q, k, v, lam, kv_in)
        ctx.group, ctx.kernels, ctx.lengths = group, kernels, lengths
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, lam, kv_in = ctx.saved_tensors
        group, kernels = ctx.group, ctx.kernels
        rank = dist.get_rank(group)
        do = do.contiguous().to(q.dtype)
        r = kernels.backward_state(q, do, lam)
        dkv_in = suffix_states(_gather(r, group), ctx.lengths, lam, rank)
        dq, dk, dv = kernels.backward(q, k, v, do, lam, kv_in, dkv_in)
        return dq, dk, dv, None, None, None, None, None


def sp_lightning_attention(q, k, v, lam, group=None, *, layout: str = "bhnd", kernels: LocalKernels | None = None,
                           lengths: Sequence[int] | None = None):
    """Sequence-parallel lightning attention over ``group`` (default: WORLD).

    ``q, k, v``: this rank's contiguous slice of positions, [b, h, n_p, d] ("bhnd") or [b, n_p, h, d]
    ("bnhd"); ranks hold slices in rank order.  ``lam``: one decay per head (float64 tensor on the
    inputs' device, or anything ``ops.decay_tensor`` accepts).  ``lengths``: every rank's slice length in
    rank order, when the caller knows them (fixed slicing); otherwise they are exchanged with one small
    all_gather per call, whose read-back synchronises the host with the stream.
    """
    if layout not in ("bhnd", "bnhd"):
        raise ShapeError(f"layout must be 'bhnd' or 'bnhd', got {layout!r}")
    group = group if group is not None else dist.group.WORLD
    heads = q.shape[1] if layout == "bhnd" else q.shape[2]
    if not isinstance(lam, torch.Tensor):
        from .ops import decay_tensor
        lam = decay_tensor(lam, heads, q.device)
    if kernels is None:
        kernels = CudaKernels(layout=layout)
    return SequenceParallelLightning.apply(q, k, v, lam, group, kernels, 2 if layout == "bhnd" else 1,
                                           None if lengths is None else [int(x) for x in lengths])
