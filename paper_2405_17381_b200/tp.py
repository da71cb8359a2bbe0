"""Tensor-parallel GLA layer with one collective (the reference's ``gla_parallel_forward``,
parallel.py:138-178, Appendix E of the paper).

Each rank owns a contiguous block of heads: the column slices of Wq, Wk, Wv, Wu for those heads
and the matching row slice of Wo (``shard_gla_weights`` = ``shard_weights``, parallel.py:97-122).
It runs its heads' attention core, gates WITHOUT the norm, multiplies its Wo rows, and appends its
attention slice's per-row sum of squares: the one all-reduce (NCCL over NVLink on GPUs) sums the
augmented [rows, d_model + 1] partials, after which the parameter-free SRMSNorm row scale is
applied from the reduced statistic -- exact, because the norm's scale is a per-row scalar that
commutes with the output projection.

The local stages are pluggable (``TpOps``): production uses the CUDA library (``CudaTpOps``);
the CPU tests plug in a torch/oracle implementation to exercise this host logic under a
world-size-2 ``gloo`` group.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Protocol

import torch
import torch.distributed as dist

from .errors import DomainError, ShapeError
from .gla import GlaWeights


class TpOps(Protocol):
    def prologue(self, qp, kp, heads, act, theta): ...
    def attention(self, q, k, v, lam, heads): ...
    def gate_rowsq(self, a, u, heads, rowsq_view, stride): ...
    def rowscale(self, red, out_width, eps): ...


class CudaTpOps:
    """The B200 library: la_gla_prologue, la_fwd (all local heads, [b, n, h, d] layout),
    la_gla_gate_rowsq, la_gla_rowscale."""

    def prologue(self, qp, kp, heads, act, theta):
        from . import ops
        return ops.gla_prologue(qp, kp, heads, act=act, theta=theta)

    def attention(self, q, k, v, lam, heads):
        from . import ops
        b, n, w = q.shape
        d = w // heads
        a = ops.la_forward(q.view(b, n, heads, d), k.view(b, n, heads, d), v.contiguous().view(b, n, heads, d), lam,
                           layout="bnhd")
        return a.view(b, n, w)

    def gate_rowsq(self, a, u, heads, rowsq_view, stride):
        from . import ops
        return ops.gla_gate_rowsq(a, u, heads, rowsq_view, rowsq_stride=stride)

    def rowscale(self, red, out_width, eps):
        from . import ops
        return ops.gla_rowscale(red, out_width, eps=eps)


@dataclass
class GlaShard:
    weights: GlaWeights  # wq, wk, wv, wu: [d_model, heads_p * d]; wo: [heads_p * d, d_model]
    head0: int           # first global head index of this shard
    heads: int           # heads on this shard


def shard_gla_weights(w: GlaWeights, heads: int, world: int) -> list[GlaShard]:
    """Head-aligned slices for ``world`` ranks (parallel.py:97-122): column slices of the input
    projections, the matching row slice of Wo.  Concatenating them restores the weights."""
    if world < 1:
        raise DomainError(f"worker count must be >= 1, got {world}")
    if heads % world:
        raise DomainError(f"heads={heads} not divisible by P={world}")
    dm = w.wq.shape[0]
    cols = dm // world
    hp = heads // world
    out = []
    for p in range(world):
        sl = slice(p * cols, (p + 1) * cols)
        out.append(GlaShard(GlaWeights(wq=w.wq[:, sl], wk=w.wk[:, sl], wv=w.wv[:, sl], wo=w.wo[sl, :],
                                       wu=w.wu[:, sl] if w.wu is not None else None), p * hp, hp))
    return out


def gla_tp_forward(x, shard: GlaShard, lam_local, group=None, *, act="swish", theta=None, eps=1e-8,
                   tp_ops: TpOps | None = None, all_reduce=None):
    """This rank's share of the layer; returns the full [batch, n, d_model] output on every rank.

    ``lam_local``: the decays of this shard's heads.  ``all_reduce`` (default
    ``torch.distributed.all_reduce`` on ``group``) is called exactly once, on the augmented
    [batch * n, d_model + 1] partials in the accumulation dtype.
    """
    ops = tp_ops if tp_ops is not None else CudaTpOps()
    w = shard.weights
    if x.dim() != 3 or x.shape[-1] != w.wq.shape[0]:
        raise ShapeError(f"x must be [batch, n, {w.wq.shape[0]}], got {tuple(x.shape)}")
    b, n, dm = x.shape
    qp, kp, v = x @ w.wq, x @ w.wk, x @ w.wv
    u = x @ w.wu if w.wu is not None else None
    q, k = ops.prologue(qp, kp, shard.heads, act, theta)
    a = ops.attention(q, k, v, lam_local, shard.heads)
    acc = torch.float64 if x.dtype == torch.float64 else torch.float32
    aug = torch.empty(b * n, dm + 1, dtype=acc, device=x.device)
    gated = ops.gate_rowsq(a, u, shard.heads, aug[:, dm], dm + 1)
    aug[:, :dm] = (gated @ w.wo).reshape(b * n, dm).to(acc)
    if all_reduce is None:
        dist.all_reduce(aug, group=group)
    else:
        all_reduce(aug)
    y = ops.rowscale(aug, dm, eps)
    return y.view(b, n, dm).to(x.dtype)
