"""The GLA token mixer of the reference's TNL model around the attention core, on the B200 path.

Reference: ``gla_forward`` / ``gla_backward`` (model.py:365-453) and the attention half of
``decode_step`` (model.py:669-709).  The reference loops over heads in Python and runs every
stage in numpy fp64; here the layer is

    y = [srmsnorm(LA(rot(act(x Wq)), rot(act(x Wk)), x Wv)) * (x Wu)] Wo

with the five projections as library GEMMs (torch / cuBLAS), the element-wise stages as the
fused CUDA kernels behind ``la_gla_*`` (one read and one write of every operand per stage), and
the attention core as one batched ``la_fwd`` / ``la_bwd`` over all heads on the model-native
[batch, n, heads, d] layout (no transposes).  Where batch * heads fills the GPU (bf16, d = 128) the
forward runs the fused core instead (``la_gla_core_fwd``: act + LRPE applied to each q / k tile in the
pass kernel's shared memory, no q / k round trip before the core).  There is no CPU fallback.

Scope: ``gla_act`` swish / one_plus_elu / none, the U gate on or off, the parameter-free
``srmsnorm`` (the reference default ``norm``); LRPE rotation when ``theta`` is given (the
reference rotates layer 1 in pe_mode "mix", every layer in "lrpe_d"; ``layer_pe_policy``,
positional.py:196-210, is the caller's choice of passing theta or not).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from ._lib import UnsupportedError
from .errors import ShapeError


class GlaCore(torch.autograd.Function):
    """gated = srmsnorm(LA(rot(act(qp)), rot(act(kp)), v)) * u on [batch, n, heads * d] rows."""

    @staticmethod
    def forward(ctx, qp, kp, v, u, theta, lam_dev, heads, act, offset, eps, backend):
        a = seg = None
        if backend in ("auto", "tcgen05"):
            # the fused core (act + LRPE in the pass kernel's load stage) where it applies
            try:
                a, q, k = ops.gla_core_forward(qp, kp, v, None, heads, act=act, theta=theta, offset=offset,
                                               lam_dev=lam_dev)
            except UnsupportedError:
                a = None
        if a is None:
            q, k = ops.gla_prologue(qp, kp, heads, act=act, theta=theta, offset=offset)
            b, n, w = q.shape
            d = w // heads
            q4, k4, v4 = (t.view(b, n, heads, d) for t in (q, k, v.contiguous()))
            a, seg = ops.la_forward(q4, k4, v4, None, layout="bnhd", backend=backend, lam_dev=lam_dev,
                                    want_seg_states=True)
            a = a.view(b, n, w)
        gated, rawnorm = ops.gla_epilogue(a, u, heads, eps=eps)
        ctx.save_for_backward(qp, kp, q, k, v, u, a, rawnorm, theta, lam_dev, seg)
        ctx.cfg = (heads, act, offset, eps, backend)
        return gated

    @staticmethod
    def backward(ctx, dgated):
        qp, kp, q, k, v, u, a, rawnorm, theta, lam_dev, seg = ctx.saved_tensors
        heads, act, offset, eps, backend = ctx.cfg
        da, du = ops.gla_epilogue_backward(dgated.to(a.dtype), a, u, rawnorm, heads, eps=eps)
        b, n, w = a.shape
        d = w // heads
        # the two-step backward: the fused one (ops.gla_core_backward, the prologue's backward on the dq / dK
        # tiles before they are stored) moves 4 rows fewer but measured 0.73-0.93x of this (K7)
        dq, dk, dv = ops.la_backward(*(t.view(b, n, heads, d) for t in (q, k, v.contiguous(), da)), None,
                                     layout="bnhd", backend=backend, lam_dev=lam_dev, fwd_seg_states=seg)
        dqp, dkp, dtheta = ops.gla_prologue_backward(qp, kp, dq.view(b, n, w), dk.view(b, n, w), heads, act=act,
                                                     theta=theta, offset=offset)
        return (dqp, dkp, dv.view(b, n, w), du, dtheta if (theta is not None and ctx.needs_input_grad[4]) else None,
                None, None, None, None, None, None)


def gla_core(qp, kp, v, u, lam, heads, *, act="swish", theta=None, offset=0, eps=ops.SRMS_EPS, backend="auto"):
    """Functional form of :class:`GlaCore`; ``lam`` holds one decay per head (frozen)."""
    lam_dev = ops.decay_tensor(lam, heads, qp.device)
    return GlaCore.apply(qp, kp, v, u, theta, lam_dev, heads, act, offset, eps, backend)


@dataclass
class GlaWeights:
    """The layer's projections, stored [d_model, d_model] like the reference's GlaWeights
    (model.py:246-262): y = x @ wq etc.  ``wu`` is None without the gate."""

    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor
    wu: torch.Tensor | None = None


def gla_forward(x, w: GlaWeights, lam, heads, *, act="swish", theta=None, offset=0, eps=ops.SRMS_EPS,
                backend="auto"):
    """The GLA layer (model.py:365-406) on x [batch, n, d_model]; differentiable in x, the
    weights and theta through torch autograd (the backward mirrors model.py:409-453)."""
    if x.dim() != 3 or x.shape[-1] != w.wq.shape[0]:
        raise ShapeError(f"x must be [batch, n, {w.wq.shape[0]}], got {tuple(x.shape)}")
    qp, kp, v = x @ w.wq, x @ w.wk, x @ w.wv
    u = x @ w.wu if w.wu is not None else None
    gated = gla_core(qp, kp, v, u, lam, heads, act=act, theta=theta, offset=offset, eps=eps, backend=backend)
    return gated @ w.wo


class DecodeState:
    """Generation state of one GLA layer: the [batch, heads, d, d] summaries and the position
    (model.py:650-667 keeps (layers, heads, d, d) for one sequence)."""

    def __init__(self, kv: torch.Tensor, position: int = 0):
        self.kv = kv
        self.position = position

    @classmethod
    def fresh(cls, batch, heads, d, dtype=torch.float32, device="cuda"):
        return cls(torch.zeros(batch, heads, d, d, dtype=ops.state_dtype(dtype), device=device), 0)

    @classmethod
    def from_prefill(cls, x, w: GlaWeights, lam, heads, *, act="swish", theta=None, eps=ops.SRMS_EPS):
        """Run the layer over a prompt x [batch, n, d_model]; returns (y, state) with state.kv =
        the forward's kv_out (the carried summary after the prompt), position = n."""
        b, n, _ = x.shape
        qp, kp, v = x @ w.wq, x @ w.wk, x @ w.wv
        u = x @ w.wu if w.wu is not None else None
        wd = qp.shape[-1]
        d = wd // heads
        try:  # the fused core; a prefill needs no q / k for a backward
            a, _, _, kv = ops.gla_core_forward(qp, kp, v, lam, heads, act=act, theta=theta, want_qk=False,
                                               want_state=True)
        except UnsupportedError:
            q, k = ops.gla_prologue(qp, kp, heads, act=act, theta=theta, offset=0)
            a, kv = ops.la_forward(q.view(b, n, heads, d), k.view(b, n, heads, d),
                                   v.contiguous().view(b, n, heads, d), lam, layout="bnhd", want_state=True)
        gated, _ = ops.gla_epilogue(a.view(b, n, wd), u, heads, eps=eps)
        return gated @ w.wo, cls(kv, n)

    def step(self, x_t, w: GlaWeights, lam, heads, *, act="swish", theta=None, eps=ops.SRMS_EPS):
        """One token per sequence, x_t [batch, d_model] -> y_t [batch, d_model]; updates the
        state in place (model.py:684-704: projections, rotation at this position, kv update,
        read-out, norm, gate, output projection)."""
        b, dm = x_t.shape
        x3 = x_t.view(b, 1, dm)
        qp, kp, v = x3 @ w.wq, x3 @ w.wk, x3 @ w.wv
        u = x3 @ w.wu if w.wu is not None else None
        q, k = ops.gla_prologue(qp, kp, heads, act=act, theta=theta, offset=self.position)
        d = dm // heads
        a = ops.la_decode(q.view(b, heads, d), k.view(b, heads, d), v.contiguous().view(b, heads, d), lam, self.kv)
        gated, _ = ops.gla_epilogue(a.reshape(b, 1, dm), u, heads, eps=eps)
        self.position += 1
        return (gated @ w.wo).view(b, dm)
