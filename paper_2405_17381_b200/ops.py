"""Batched device entry points: torch CUDA tensors in, torch CUDA tensors out.

These are thin host wrappers over the C ABI (``_lib``): they validate like
the reference (``AttentionConfig`` / ``_prep``, kernels.py:84-150), build the
``la_desc``, allocate outputs and workspace with torch's caching allocator,
and launch on the current stream.  Nothing here computes on the CPU.

Tensor layouts: ``"bhnd"`` = [batch, heads, n, d] (default) or ``"bnhd"`` =
[batch, n, heads, d] (the model-native projection layout; no transpose copy).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib
from .errors import DomainError, ShapeError, check_decay

_DTYPES = {torch.float32: _lib.LA_F32, torch.float64: _lib.LA_F64, torch.bfloat16: _lib.LA_BF16}


def state_dtype(dtype: torch.dtype) -> torch.dtype:
    """Carried-state dtype: fp64 for the fp64 path, fp32 otherwise."""
    return torch.float64 if dtype == torch.float64 else torch.float32


_DECAY_CACHE: dict = {}
_DECAY_CACHE_MAX = 64


def decay_tensor(lam, heads: int, device) -> torch.Tensor:
    """Validate per-head decays (host side) and return a device fp64 [heads] tensor.

    Results are cached per (values, device): a call with host values (float / list / CPU tensor)
    after the first costs no host-to-device copy, so the autograd ops and the GLA layer keep the
    host ahead of the GPU (a pageable copy per call would serialise them) and stay capturable in a
    CUDA graph.  The returned tensor is shared: treat it as read-only.  A CUDA tensor argument is
    read back to validate it (a synchronisation) -- build it once with this function instead."""
    if isinstance(lam, torch.Tensor):
        vals = lam.detach().to("cpu", torch.float64).reshape(-1).tolist()
    elif isinstance(lam, (int, float)):
        vals = [float(lam)] * heads
    else:
        vals = [float(x) for x in lam]
    if len(vals) == 1 and heads > 1:
        vals = vals * heads
    if len(vals) != heads:
        raise ShapeError(f"need one decay per head: got {len(vals)} for {heads} heads")
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (tuple(vals), dev.type, dev.index)
    hit = _DECAY_CACHE.get(key)
    if hit is not None:
        return hit
    for x in vals:
        check_decay(x)
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if len(_DECAY_CACHE) >= _DECAY_CACHE_MAX:
        _DECAY_CACHE.pop(next(iter(_DECAY_CACHE)))
    _DECAY_CACHE[key] = t
    return t


@dataclass(frozen=True)
class Geometry:
    batch: int
    heads: int
    n: int
    d: int
    strides: tuple[int, int, int]


def _geometry(x: torch.Tensor, layout: str) -> Geometry:
    if x.dim() != 4:
        raise ShapeError(f"expected a 4-D tensor ({layout}), got shape {tuple(x.shape)}")
    if layout == "bhnd":
        b, h, n, d = x.shape
        s = (x.stride(0), x.stride(1), x.stride(2))
    elif layout == "bnhd":
        b, n, h, d = x.shape
        s = (x.stride(0), x.stride(2), x.stride(1))
    else:
        raise DomainError(f"layout must be 'bhnd' or 'bnhd', got {layout!r}")
    return Geometry(b, h, n, d, s)


def _tc_ready(t: torch.Tensor, layout: str) -> bool:
    """TMA-describable on the tensor-core path: 16-byte aligned base and (batch, head, position) strides."""
    return t.data_ptr() % 16 == 0 and all((x * t.element_size()) % 16 == 0 for x in _geometry(t, layout).strides)


def _prep(tensors: Sequence[torch.Tensor], names: str, layout: str):
    """Shape/dtype/device checks (the reference's _prep, kernels.py:133-150, minus its copy-cast).

    Each operand keeps its own strides (la_tensor_strides): a view with a unit feature stride is
    passed as is.  A copy is made only when the kernels cannot address the view -- a feature
    stride != 1, or, for bf16 / fp32 operands at d = 32, 64, 96 or 128 (the tensor-core paths), a
    base or stride that is no multiple of 16 bytes -- and then only of that operand."""
    first = tensors[0]
    if not isinstance(first, torch.Tensor):
        raise ShapeError(f"{names[0]}: expected a torch.Tensor")
    if first.dtype not in _DTYPES:
        raise DomainError(f"dtype must be float32, float64 or bfloat16, got {first.dtype}")
    if not first.is_cuda:
        raise DomainError(f"{names[0]}: tensors must live on a CUDA device (no CPU path)")
    for t, name in zip(tensors, names):
        if not isinstance(t, torch.Tensor):
            raise ShapeError(f"{name}: expected a torch.Tensor")
        if t.shape != first.shape:
            raise ShapeError(f"{name}: shape {tuple(t.shape)} != {tuple(first.shape)}")
        if t.dtype != first.dtype or t.device != first.device:
            raise ShapeError(f"{name}: dtype/device {t.dtype}/{t.device} != {first.dtype}/{first.device}")
    g = _geometry(first, layout)
    tc = first.dtype in (torch.bfloat16, torch.float32) and g.d % 32 == 0 and g.d <= 128
    out = []
    for t in tensors:
        if t.dim() == 4 and t.stride(3) != 1 and t.shape[3] > 1:
            t = t.contiguous()
        if tc and not _tc_ready(t, layout):
            t = t.contiguous() if not t.is_contiguous() else t.clone()  # clone: a fresh, aligned base
        out.append(t)
    return out, _geometry(out[0], layout)


def _strides(layout: str, pairs) -> _lib.LaTensorStrides:
    """la_tensor_strides from (operand index, tensor) pairs."""
    st = _lib.LaTensorStrides()
    for idx, t in pairs:
        if t is None:
            continue
        sg = _geometry(t, layout).strides
        for j in range(3):
            st.s[idx][j] = sg[j]
    return st


def _out(g: Geometry, like: torch.Tensor, layout: str) -> torch.Tensor:
    """A fresh contiguous output in the call's layout."""
    shape = (g.batch, g.heads, g.n, g.d) if layout == "bhnd" else (g.batch, g.n, g.heads, g.d)
    return torch.empty(shape, dtype=like.dtype, device=like.device)


def _desc(g: Geometry, dtype: torch.dtype, block, backend: str, segments: int) -> _lib.LaDesc:
    if block is not None and int(block) < 1:
        raise DomainError(f"block size must be >= 1, got {block}")
    if backend not in _lib.BACKENDS:
        raise DomainError(f"backend must be one of {sorted(_lib.BACKENDS)}, got {backend!r}")
    desc = _lib.LaDesc()
    desc.batch, desc.heads, desc.n, desc.d = g.batch, g.heads, g.n, g.d
    desc.block = 0 if block is None else int(block)
    desc.dtype = _DTYPES[dtype]
    desc.backend = _lib.BACKENDS[backend]
    for i in range(3):
        desc.stride[i] = g.strides[i]
    desc.segments = int(segments)
    return desc


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _lam_ptr(lam_dev: torch.Tensor, heads: int, device):
    """The device decay array the kernels read: must be a contiguous float64 CUDA tensor of `heads`
    values on the operands' device (decay_tensor builds one); anything else would be misread."""
    dev = torch.device(device)
    if (not isinstance(lam_dev, torch.Tensor) or lam_dev.dtype != torch.float64 or not lam_dev.is_cuda
            or lam_dev.numel() != heads or not lam_dev.is_contiguous()
            or (dev.index is not None and lam_dev.device != dev)):
        raise ShapeError(f"lam_dev must be a contiguous float64 CUDA tensor of {heads} values on {device} "
                         f"(use ops.decay_tensor), got {getattr(lam_dev, 'dtype', type(lam_dev))} "
                         f"{tuple(getattr(lam_dev, 'shape', ()))} on {getattr(lam_dev, 'device', '?')}")
    return ctypes.cast(ctypes.c_void_p(lam_dev.data_ptr()), ctypes.POINTER(ctypes.c_double))


def _lam(lam, lam_dev, heads, device):
    """(device decay tensor, its pointer): lam_dev as given (validated) or built from host values."""
    if lam_dev is None:
        lam_dev = decay_tensor(lam, heads, device)
    return lam_dev, _lam_ptr(lam_dev, heads, device)


def _state(t, g: Geometry, dtype, name):
    if t is None:
        return None
    if t.shape != (g.batch, g.heads, g.d, g.d):
        raise ShapeError(f"{name}: expected shape {(g.batch, g.heads, g.d, g.d)}, got {tuple(t.shape)}")
    t = t.to(dtype=state_dtype(dtype)).contiguous()
    return t if t.data_ptr() % 16 == 0 else t.clone()  # the kernels read state rows as 16-byte vectors


def _workspace(lib, desc, device, workspace=None):
    nbytes = lib.la_workspace_bytes(ctypes.byref(desc))
    if workspace is not None:
        if workspace.device != torch.device(device) or workspace.numel() * workspace.element_size() < nbytes:
            raise ShapeError(f"workspace: need {nbytes} bytes on {device}")
        return workspace, workspace.numel() * workspace.element_size()
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
    return ws, nbytes


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(device) -> ctypes.c_void_p:
    # the raw handle of the caller's current stream; torch.cuda.current_stream() builds a Stream
    # object per call (~7 us of a ~25 us host path for a decode step)
    if _RAW_STREAM is not None:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        return ctypes.c_void_p(_RAW_STREAM(idx))
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def segment_count(desc) -> int:
    return int(_lib.load().la_segment_count(ctypes.byref(desc)))


def _flags(check: bool, resume: bool) -> int:
    f = _lib.LA_FLAG_RESUME if resume else 0
    if check:
        f |= _lib.LA_FLAG_CHECK_DECAY | _lib.LA_FLAG_CHECK_FINITE
    return f


def la_forward(q, k, v, lam, *, block=None, kv_in=None, want_state=False, layout="bhnd",
               backend="auto", segments=0, lam_dev=None, want_seg_states=False, check=False, workspace=None,
               resume=False):
    """o (and kv_out) for batched q, k, v.  ``lam``: float or one value per head.

    ``want_seg_states``: also return the state entering every sequence segment (or None when the
    library does not split the sequence) -- pass it to ``la_backward(fwd_seg_states=...)``.
    ``check``: validate lam and scan q, k, v for NaN / Inf on the device (synchronises; the reference
    always does both, kernels.py:84-91,148-149).  ``resume`` (with ``workspace``): the workspace holds
    ``la_forward_state(k, v, ..., workspace=...)``'s summaries for this problem, so the summary pass is
    skipped (sequence parallelism).
    """
    (q, k, v), g = _prep([q, k, v], "QKV", layout)
    lib = _lib.load()
    desc = _desc(g, q.dtype, block, backend, segments)
    lam_dev, lam_p = _lam(lam, lam_dev, g.heads, q.device)
    kv_in = _state(kv_in, g, q.dtype, "kv_in")
    o = _out(g, q, layout)
    kv_out = torch.empty((g.batch, g.heads, g.d, g.d), dtype=state_dtype(q.dtype), device=q.device) \
        if want_state else None
    seg = None
    if want_seg_states:
        nseg = segment_count(desc)
        if nseg > 1:
            seg = torch.empty((g.batch, g.heads, nseg, g.d, g.d), dtype=state_dtype(q.dtype), device=q.device)
    if resume and workspace is None:
        raise ShapeError("resume=True needs the workspace la_forward_state filled")
    ws, nbytes = _workspace(lib, desc, q.device, workspace)
    st = _strides(layout, ((_lib.LA_T_Q, q), (_lib.LA_T_K, k), (_lib.LA_T_V, v), (_lib.LA_T_O, o)))
    _lib.check(lib.la_fwd_ex(ctypes.byref(desc), ctypes.byref(st), _flags(check, resume), _ptr(q), _ptr(k), _ptr(v),
                             lam_p, _ptr(kv_in), _ptr(o), _ptr(kv_out), _ptr(seg), _ptr(ws), nbytes,
                             _stream(q.device)))
    out = (o, kv_out) if want_state else o
    return (out, seg) if want_seg_states else out


_PARTS = {"all": 0, "dq": _lib.LA_FLAG_NO_DKDV, "dkdv": _lib.LA_FLAG_NO_DQ}


def la_backward(q, k, v, do, lam, *, block=None, kv_in=None, dkv_in=None, want_state=False, layout="bhnd",
                backend="auto", segments=0, lam_dev=None, fwd_seg_states=None, check=False, parts="all",
                workspace=None, resume=False):
    """(dq, dk, dv) (and dkv_out = R(0)) of <LA(q, k, v), do>.

    ``fwd_seg_states``: the forward's segment states for the same problem and kv_in (optional).
    ``parts``: "all", "dq" (sweep 1 only; dk, dv come back None) or "dkdv" (sweep 2 only; dq None).
    ``resume`` (with ``workspace``): the workspace holds ``la_backward_state(q, do, ...,
    workspace=...)``'s adjoint summaries, so sweep 2 skips its summary pass.
    """
    if parts not in _PARTS:
        raise DomainError(f"parts must be one of {sorted(_PARTS)}, got {parts!r}")
    (q, k, v, do), g = _prep([q, k, v, do], ["Q", "K", "V", "dO"], layout)
    lib = _lib.load()
    desc = _desc(g, q.dtype, block, backend, segments)
    lam_dev, lam_p = _lam(lam, lam_dev, g.heads, q.device)
    kv_in = _state(kv_in, g, q.dtype, "kv_in")
    dkv_in = _state(dkv_in, g, q.dtype, "dkv_in")
    dq = _out(g, q, layout) if parts != "dkdv" else None
    dk, dv = (_out(g, q, layout), _out(g, q, layout)) if parts != "dq" else (None, None)
    dkv_out = torch.empty((g.batch, g.heads, g.d, g.d), dtype=state_dtype(q.dtype), device=q.device) \
        if (want_state and parts != "dq") else None
    if resume and workspace is None:
        raise ShapeError("resume=True needs the workspace la_backward_state filled")
    ws, nbytes = _workspace(lib, desc, q.device, workspace)
    if fwd_seg_states is not None:
        want = (g.batch, g.heads, segment_count(desc), g.d, g.d)
        if tuple(fwd_seg_states.shape) != want:
            raise ShapeError(f"fwd_seg_states has shape {tuple(fwd_seg_states.shape)}, this problem's plan "
                             f"needs {want}")
        if fwd_seg_states.dtype != state_dtype(q.dtype) or fwd_seg_states.device != q.device \
                or not fwd_seg_states.is_contiguous():
            raise ShapeError(f"fwd_seg_states must be a contiguous {state_dtype(q.dtype)} tensor on {q.device}")
    st = _strides(layout, ((_lib.LA_T_Q, q), (_lib.LA_T_K, k), (_lib.LA_T_V, v), (_lib.LA_T_DO, do),
                           (_lib.LA_T_DQ, dq), (_lib.LA_T_DK, dk), (_lib.LA_T_DV, dv)))
    _lib.check(lib.la_bwd_ex(ctypes.byref(desc), ctypes.byref(st), _flags(check, resume) | _PARTS[parts], _ptr(q),
                             _ptr(k), _ptr(v), _ptr(do), lam_p, _ptr(kv_in), _ptr(dkv_in), _ptr(fwd_seg_states),
                             _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dkv_out), _ptr(ws), nbytes, _stream(q.device)))
    return (dq, dk, dv, dkv_out) if want_state else (dq, dk, dv)


def new_workspace(shape, dtype=torch.bfloat16, *, layout="bhnd", backend="auto", segments=0, device="cuda"):
    """A workspace for ``la_forward_state`` -> ``la_forward(resume=True)`` (or the backward pair)."""
    return torch.empty(max(workspace_bytes(shape, dtype, layout=layout, backend=backend, segments=segments), 1),
                       dtype=torch.uint8, device=device)


def la_forward_state(k, v, lam, *, layout="bhnd", backend="auto", segments=0, lam_dev=None, workspace=None):
    """Local forward summary sum_s lam^(n-1-s) k_s v_s^T, [batch, heads, d, d].  With ``workspace``
    the per-segment summaries stay there for ``la_forward(..., workspace=..., resume=True)``."""
    (k, v), g = _prep([k, v], "KV", layout)
    if _geometry(v, layout).strides != g.strides:  # la_fwd_state addresses both with the desc's strides
        k, v = k.contiguous(), v.contiguous()
        g = _geometry(k, layout)
    lib = _lib.load()
    desc = _desc(g, k.dtype, None, backend, segments)
    lam_dev, lam_p = _lam(lam, lam_dev, g.heads, k.device)
    out = torch.empty((g.batch, g.heads, g.d, g.d), dtype=state_dtype(k.dtype), device=k.device)
    ws, nbytes = _workspace(lib, desc, k.device, workspace)
    _lib.check(lib.la_fwd_state(ctypes.byref(desc), _ptr(k), _ptr(v), lam_p, _ptr(out), _ptr(ws),
                                nbytes, _stream(k.device)))
    return out


def la_backward_state(q, do, lam, *, layout="bhnd", backend="auto", segments=0, lam_dev=None, workspace=None):
    """Local adjoint summary sum_t lam^(t+1) q_t do_t^T, [batch, heads, d, d].  With ``workspace`` the
    per-segment summaries stay there for ``la_backward(..., workspace=..., resume=True)``."""
    (q, do), g = _prep([q, do], ["Q", "dO"], layout)
    if _geometry(do, layout).strides != g.strides:  # la_bwd_state addresses both with the desc's strides
        q, do = q.contiguous(), do.contiguous()
        g = _geometry(q, layout)
    lib = _lib.load()
    desc = _desc(g, q.dtype, None, backend, segments)
    lam_dev, lam_p = _lam(lam, lam_dev, g.heads, q.device)
    out = torch.empty((g.batch, g.heads, g.d, g.d), dtype=state_dtype(q.dtype), device=q.device)
    ws, nbytes = _workspace(lib, desc, q.device, workspace)
    _lib.check(lib.la_bwd_state(ctypes.byref(desc), _ptr(q), _ptr(do), lam_p, _ptr(out), _ptr(ws),
                                nbytes, _stream(q.device)))
    return out


def workspace_bytes(shape, dtype=torch.bfloat16, *, layout="bhnd", backend="auto", segments=0) -> int:
    """la_workspace_bytes for a [b, h, n, d] (or bnhd) problem, without tensors."""
    if layout == "bhnd":
        b, h, n, d = shape
        strides = (h * n * d, n * d, d)
    else:
        b, n, h, d = shape
        strides = (n * h * d, d, h * d)
    desc = _desc(Geometry(b, h, n, d, strides), dtype, None, backend, segments)
    return int(_lib.load().la_workspace_bytes(ctypes.byref(desc)))


def launch_count(shape, dtype=torch.bfloat16, *, which="fwd", layout="bhnd", backend="auto", segments=0) -> int:
    """Kernels one call launches for this problem (la_launch_count): which = "fwd", "bwd", or
    "bwd_saved" (backward given the forward's segment states)."""
    if layout == "bhnd":
        b, h, n, d = shape
        strides = (h * n * d, n * d, d)
    else:
        b, n, h, d = shape
        strides = (n * h * d, d, h * d)
    desc = _desc(Geometry(b, h, n, d, strides), dtype, None, backend, segments)
    return int(_lib.load().la_launch_count(ctypes.byref(desc), {"fwd": 0, "bwd": 1, "bwd_saved": 2}[which]))


# ----------------------------------------------------------------------------------------------
# Recurrent decode (model.py:669-709) and the GLA layer stages around the core (model.py:365-453)


def la_decode(q, k, v, lam, kv, *, lam_dev=None):
    """One decode step for every (batch, head): ``kv <- lam kv + k v^T`` in place, returns
    ``o = q . kv`` (model.py:697-701).  q, k, v: [batch, heads, d]; kv: [batch, heads, d, d] in the
    state dtype (fp32, or fp64 for fp64 operands), e.g. la_forward's kv_out after a prefill."""
    for t, name in ((q, "Q"), (k, "K"), (v, "V")):
        if not isinstance(t, torch.Tensor) or t.dim() != 3:
            raise ShapeError(f"{name}: expected a [batch, heads, d] tensor")
    # la_decode addresses q, k, v and o with the desc's one (batch, head) stride pair: one dense layout
    (q4, k4, v4), g = _prep([q.contiguous().unsqueeze(2), k.contiguous().unsqueeze(2), v.contiguous().unsqueeze(2)],
                            "QKV", "bhnd")
    if not isinstance(kv, torch.Tensor) or kv.shape != (g.batch, g.heads, g.d, g.d):
        raise ShapeError(f"kv: expected shape {(g.batch, g.heads, g.d, g.d)}")
    if kv.dtype != state_dtype(q.dtype) or not kv.is_contiguous() or kv.device != q.device:
        raise ShapeError(f"kv: expected a contiguous {state_dtype(q.dtype)} tensor on {q.device} (updated in place)")
    lib = _lib.load()
    desc = _desc(g, q4.dtype, None, "auto", 0)
    lam_dev, lam_p = _lam(lam, lam_dev, g.heads, q.device)
    o = torch.empty_like(q4)
    _lib.check(lib.la_decode(ctypes.byref(desc), _ptr(q4), _ptr(k4), _ptr(v4), lam_p, _ptr(kv), _ptr(o),
                             _stream(q.device)))
    return o.squeeze(2)


SRMS_EPS = 1e-8  # model.py:48


def _gla_desc(x: torch.Tensor, heads: int, act: str, offset: int, eps: float) -> _lib.LaGlaDesc:
    if x.dim() != 3:
        raise ShapeError(f"expected a [batch, n, heads * d] tensor, got shape {tuple(x.shape)}")
    if x.dtype not in _DTYPES:
        raise DomainError(f"dtype must be float32, float64 or bfloat16, got {x.dtype}")
    if not x.is_cuda:
        raise DomainError("tensors must live on a CUDA device (no CPU path)")
    if act not in _lib.ACTS:
        raise DomainError(f"act must be one of {sorted(_lib.ACTS)}, got {act!r}")
    b, n, w = x.shape
    if heads < 1 or w % heads:
        raise ShapeError(f"width {w} not divisible by heads={heads}")
    desc = _lib.LaGlaDesc()
    desc.batch, desc.n, desc.heads, desc.d = b, n, heads, w // heads
    desc.dtype = _DTYPES[x.dtype]
    desc.act = _lib.ACTS[act]
    desc.offset = int(offset)
    desc.eps = float(eps)
    return desc


def _rows(tensors, names):
    first = tensors[0]
    out = []
    for t, name in zip(tensors, names):
        if t is None:
            out.append(None)
            continue
        if t.shape != first.shape or t.dtype != first.dtype or t.device != first.device:
            raise ShapeError(f"{name}: shape/dtype/device {tuple(t.shape)}/{t.dtype}/{t.device} do not match "
                             f"{tuple(first.shape)}/{first.dtype}/{first.device}")
        t = t.contiguous()
        out.append(t if t.data_ptr() % 16 == 0 else t.clone())  # the stages move 16-byte vectors
    return out


def _theta(theta, d, device):
    if theta is None:
        return None
    th = torch.as_tensor(theta, dtype=torch.float64).to(device).contiguous()
    if th.shape != (d // 2,):
        raise ShapeError(f"theta has shape {tuple(th.shape)}, expected ({d // 2},)")
    return th


def gla_prologue(qp, kp, heads, *, act="swish", theta=None, offset=0):
    """q = rot(act(qp)), k = rot(act(kp)) on [batch, n, heads * d] rows (model.py:381-392)."""
    qp, kp = _rows([qp, kp], ["qp", "kp"])
    desc = _gla_desc(qp, heads, act, offset, SRMS_EPS)
    th = _theta(theta, desc.d, qp.device)
    q, k = torch.empty_like(qp), torch.empty_like(kp)
    _lib.check(_lib.load().la_gla_prologue(ctypes.byref(desc), _ptr(qp), _ptr(kp), _ptr(th), _ptr(q), _ptr(k),
                                           _stream(qp.device)))
    return q, k


def gla_core_forward(qp, kp, v, lam, heads, *, act="swish", theta=None, offset=0, lam_dev=None, want_qk=True,
                     kv_in=None, want_state=False):
    """The fused GLA core forward (la_gla_core_fwd): o = LA(rot(act(qp)), rot(act(kp)), v) on
    [batch, n, heads * d] rows in one tensor-core pass, the prologue applied to each tile in shared
    memory.  Returns (o, q, k[, kv_out]) -- q, k the transformed rows for the backward (None when
    ``want_qk`` is False).  Split sequences (batch * heads too small to fill the GPU) run the summary pass with
    the prologue too.  Raises UnsupportedError where the fused pass does not apply (not bf16 / d = 128):
    ``gla_prologue`` + ``la_forward`` compute the same thing there."""
    qp, kp, v = _rows([qp, kp, v], ["qp", "kp", "v"])
    desc = _gla_desc(qp, heads, act, offset, SRMS_EPS)
    th = _theta(theta, desc.d, qp.device)
    lam_dev, lam_p = _lam(lam, lam_dev, heads, qp.device)
    g = Geometry(desc.batch, heads, desc.n, desc.d, None)
    kv_in = _state(kv_in, g, qp.dtype, "kv_in")
    o = torch.empty_like(qp)
    q, k = (torch.empty_like(qp), torch.empty_like(kp)) if want_qk else (None, None)
    kv_out = torch.empty((desc.batch, heads, desc.d, desc.d), dtype=state_dtype(qp.dtype), device=qp.device) \
        if want_state else None
    lib = _lib.load()
    nbytes = lib.la_gla_core_workspace_bytes(ctypes.byref(desc))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=qp.device) if nbytes else None
    _lib.check(lib.la_gla_core_fwd(ctypes.byref(desc), _ptr(qp), _ptr(kp), _ptr(v), lam_p, _ptr(th), _ptr(kv_in),
                                   _ptr(o), _ptr(q), _ptr(k), _ptr(kv_out), _ptr(ws), nbytes, _stream(qp.device)))
    return (o, q, k, kv_out) if want_state else (o, q, k)


def gla_core_backward(qp, kp, q, k, v, da, lam, heads, *, act="swish", theta=None, offset=0, lam_dev=None,
                      kv_in=None, dkv_in=None, want_state=False):
    """The fused GLA core backward (la_gla_core_bwd): (dqp, dkp, dv) of the core on [batch, n, heads * d] rows --
    the core's backward on the forward's q, k (``gla_core_forward``'s q / k out), v and da, with the prologue's
    backward (act' and the inverse LRPE rotation) applied to the dq / dK tiles before they are stored.  No angle
    gradient (use ``la_backward`` + ``gla_prologue_backward`` when theta is learned).  Raises UnsupportedError
    outside bf16 / d = 128."""
    qp, kp, q, k, v, da = _rows([qp, kp, q, k, v, da], ["qp", "kp", "q", "k", "v", "da"])
    desc = _gla_desc(qp, heads, act, offset, SRMS_EPS)
    th = _theta(theta, desc.d, qp.device)
    lam_dev, lam_p = _lam(lam, lam_dev, heads, qp.device)
    g = Geometry(desc.batch, heads, desc.n, desc.d, None)
    kv_in = _state(kv_in, g, qp.dtype, "kv_in")
    dkv_in = _state(dkv_in, g, qp.dtype, "dkv_in")
    dqp, dkp, dv = torch.empty_like(qp), torch.empty_like(kp), torch.empty_like(v)
    dkv_out = torch.empty((desc.batch, heads, desc.d, desc.d), dtype=state_dtype(qp.dtype), device=qp.device) \
        if want_state else None
    lib = _lib.load()
    nbytes = lib.la_gla_core_bwd_workspace_bytes(ctypes.byref(desc))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=qp.device) if nbytes else None
    _lib.check(lib.la_gla_core_bwd(ctypes.byref(desc), _ptr(qp), _ptr(kp), _ptr(q), _ptr(k), _ptr(v), _ptr(da), lam_p,
                                   _ptr(th), _ptr(kv_in), _ptr(dkv_in), _ptr(dqp), _ptr(dkp), _ptr(dv), _ptr(dkv_out),
                                   _ptr(ws), nbytes, _stream(qp.device)))
    return (dqp, dkp, dv, dkv_out) if want_state else (dqp, dkp, dv)


def gla_prologue_backward(qp, kp, dq, dk, heads, *, act="swish", theta=None, offset=0, dtheta=None):
    """(dqp, dkp) of gla_prologue; with theta, the angle gradient is accumulated into ``dtheta``
    (fp64 [d/2], created when None) and returned as the third value."""
    qp, kp, dq, dk = _rows([qp, kp, dq, dk], ["qp", "kp", "dq", "dk"])
    desc = _gla_desc(qp, heads, act, offset, SRMS_EPS)
    lib = _lib.load()
    th = _theta(theta, desc.d, qp.device)
    if th is not None and dtheta is None:
        dtheta = torch.zeros(desc.d // 2, dtype=torch.float64, device=qp.device)
    nbytes = lib.la_gla_workspace_bytes(ctypes.byref(desc)) if th is not None else 0
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=qp.device)
    dqp, dkp = torch.empty_like(qp), torch.empty_like(kp)
    _lib.check(lib.la_gla_prologue_bwd(ctypes.byref(desc), _ptr(qp), _ptr(kp), _ptr(th), _ptr(dq), _ptr(dk),
                                       _ptr(dqp), _ptr(dkp), _ptr(dtheta if th is not None else None), _ptr(ws),
                                       nbytes, _stream(qp.device)))
    return dqp, dkp, (dtheta if th is not None else None)


def gla_epilogue(a, u, heads, *, eps=SRMS_EPS):
    """gated = srmsnorm(a) * u (u None: no gate) over each row; returns (gated, rawnorm)."""
    a, u = _rows([a, u], ["a", "u"])
    desc = _gla_desc(a, heads, "none", 0, eps)
    gated = torch.empty_like(a)
    rawnorm = torch.empty(a.shape[0] * a.shape[1], dtype=state_dtype(a.dtype), device=a.device)
    _lib.check(_lib.load().la_gla_epilogue(ctypes.byref(desc), _ptr(a), _ptr(u), _ptr(gated), _ptr(rawnorm),
                                           _stream(a.device)))
    return gated, rawnorm


def gla_epilogue_backward(dgated, a, u, rawnorm, heads, *, eps=SRMS_EPS):
    """(da, du) of gla_epilogue (du None when u is None)."""
    dgated, a, u = _rows([dgated, a, u], ["dgated", "a", "u"])
    desc = _gla_desc(a, heads, "none", 0, eps)
    da = torch.empty_like(a)
    du = torch.empty_like(a) if u is not None else None
    _lib.check(_lib.load().la_gla_epilogue_bwd(ctypes.byref(desc), _ptr(dgated), _ptr(a), _ptr(u),
                                               _ptr(rawnorm.contiguous()), _ptr(da), _ptr(du), _stream(a.device)))
    return da, du


def gla_gate_rowsq(a, u, heads, rowsq, *, rowsq_stride=1):
    """Tensor-parallel stage: gated = a * u (u None: a copy of a) and rowsq[r * stride] = |a_r|^2
    written into ``rowsq`` (a view into the all-reduce buffer, accumulation dtype)."""
    a, u = _rows([a, u], ["a", "u"])
    desc = _gla_desc(a, heads, "none", 0, SRMS_EPS)
    if rowsq.dtype != state_dtype(a.dtype) or rowsq.device != a.device:
        raise ShapeError(f"rowsq must be {state_dtype(a.dtype)} on {a.device}")
    gated = torch.empty_like(a)
    _lib.check(_lib.load().la_gla_gate_rowsq(ctypes.byref(desc), _ptr(a), _ptr(u), _ptr(gated), _ptr(rowsq),
                                             int(rowsq_stride), _stream(a.device)))
    return gated


def gla_rowscale(red, out_width, *, eps=SRMS_EPS, dtype=torch.float32):
    """y[r, :] = red[r, :W] sqrt(W) / max(sqrt(red[r, W]), eps) on the reduced [rows, W + 1] buffer."""
    if red.dim() != 2 or red.shape[1] != out_width + 1 or red.dtype not in (torch.float32, torch.float64):
        raise ShapeError(f"red must be a float32/float64 [rows, {out_width + 1}] tensor, got {tuple(red.shape)} "
                         f"{red.dtype}")
    red = red.contiguous()
    y = torch.empty(red.shape[0], out_width, dtype=red.dtype, device=red.device)
    code = _lib.LA_F64 if red.dtype == torch.float64 else _lib.LA_F32
    _lib.check(_lib.load().la_gla_rowscale(code, red.shape[0], out_width, float(eps), _ptr(red), _ptr(y),
                                           _stream(red.device)))
    return y
