"""``torch.autograd.Function`` drop-in for the reference's per-head kernel calls.

The reference's model calls ``lightning_forward_decay`` / ``lightning_backward_decay``
once per head in a Python loop (model.py:393-401, 432-442).  Here one call
covers every (batch, head): q, k, v are [batch, heads, n, d] (or the
model-native [batch, n, heads, d] with ``layout="bnhd"``) and ``lam`` holds
one frozen decay per head (no gradient).  Forward saves q, k, v
only; the backward recomputes the carried state, as the reference does
(kernels.py:309-318).
"""

from __future__ import annotations

import torch

from . import ops


class LightningAttention(torch.autograd.Function):
    """o = LA(q, k, v; lam) with exact causal decayed linear attention."""

    @staticmethod
    def forward(ctx, q, k, v, lam, block=None, layout="bhnd", backend="auto"):
        heads = q.shape[1] if layout == "bhnd" else q.shape[2]
        # a device decay array is used as is only when it already is what the kernels read (one contiguous
        # fp64 value per head on q's device; a value outside (0, 1] comes back as NaN outputs, load_decay);
        # anything else -- host values, a broadcast scalar, another dtype or device -- goes through the
        # validated, cached decay_tensor
        fast = (isinstance(lam, torch.Tensor) and lam.is_cuda and lam.dtype == torch.float64
                and lam.numel() == heads and lam.is_contiguous() and lam.device == q.device)
        lam_dev = lam if fast else ops.decay_tensor(lam, heads, q.device)
        o, seg = ops.la_forward(q, k, v, None, block=block, layout=layout, backend=backend, lam_dev=lam_dev,
                                want_seg_states=True)
        # the per-segment states of a split sequence spare the backward one summary pass (la_bwd)
        ctx.save_for_backward(q, k, v, lam_dev, seg)
        ctx.block, ctx.layout, ctx.backend = block, layout, backend
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, lam_dev, seg = ctx.saved_tensors
        dq, dk, dv = ops.la_backward(q, k, v, do.to(q.dtype), None, block=ctx.block, layout=ctx.layout,
                                     backend=ctx.backend, lam_dev=lam_dev, fwd_seg_states=seg)
        return dq, dk, dv, None, None, None, None


def lightning_attention(q, k, v, lam, block=None, layout="bhnd", backend="auto"):
    """Functional form of :class:`LightningAttention`."""
    return LightningAttention.apply(q, k, v, lam, block, layout, backend)
