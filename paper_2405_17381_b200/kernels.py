"""Reference-compatible adapter: the ``linattn.kernels`` call surface on the GPU.

Same names, argument meaning and error behaviour as the reference
(kernels.py:64-471), so its tests and harness can be re-pointed here:

    AttentionConfig(n, d, B=None, lam=1.0, precision="reference")   kernels.py:69-105
    lightning_forward(q, k, v, cfg)          -> ndarray              kernels.py:158-183
    lightning_backward(q, k, v, do, cfg)     -> GradBundle           kernels.py:186-231
    lightning_forward_decay(q, k, v, cfg)    -> ndarray              kernels.py:253-284
    lightning_backward_decay(q, k, v, do, cfg) -> GradBundle         kernels.py:287-334
    KvState, GradBundle, TimingRecord, bench_kernel, aux_state_bytes
    KERNEL_KINDS = ("left", "right", "lightning", "lightning-decay")  kernels.py:64

The "left" / "right" kinds of the timing harness (Fig. 1/2 of the paper) are the reference's
float64 baselines (oracles.py:100-162), run on the device: "left" is the quadratic left product
[(Q K^T) * M] V with cuBLAS GEMMs (and its materialised-score backward), "right" the per-token
recurrence kv_t = lam kv_(t-1) + k_t v_t^T as one la_decode launch per position (its backward, the
two sequential sweeps of reference_backward, as three such walks).

Inputs are 2-D host arrays (one head), as in the reference; they are copied
to the current CUDA device, computed by the CUDA library (fp64 kernels for
precision="reference", fp32 for "working", and -- an extension -- bf16
operands with fp32 accumulation for "bf16"), and copied back.  There is no
CPU compute path: without a GPU or the built library these raise.
"""

from __future__ import annotations

from dataclasses import dataclass
from statistics import median

import numpy as np
import torch

from . import ops
from .errors import DomainError, ShapeError, check_decay

KERNEL_KINDS = ("left", "right", "lightning", "lightning-decay")

_PRECISIONS = {"working": np.float32, "reference": np.float64, "bf16": np.float32}
_TORCH = {"working": torch.float32, "reference": torch.float64, "bf16": torch.bfloat16}


@dataclass(frozen=True)
class AttentionConfig:
    """Shape, block size, decay and precision for one attention call (kernels.py:69-105)."""

    n: int
    d: int
    B: int | None = None
    lam: float = 1.0
    precision: str = "reference"

    def __post_init__(self):
        if self.n < 1 or self.d < 1:
            raise DomainError(f"need n >= 1 and d >= 1, got n={self.n}, d={self.d}")
        check_decay(self.lam)
        if self.precision not in _PRECISIONS:
            raise DomainError(f"precision must be one of {sorted(_PRECISIONS)}")
        if self.B is not None and self.B < 1:
            raise DomainError(f"block size must be >= 1, got {self.B}")

    @property
    def block(self) -> int:
        """Effective block size: default min(d, n), clamped to [1, n] (kernels.py:93-97)."""
        b = min(self.d, self.n) if self.B is None else self.B
        return max(1, min(b, self.n))

    @property
    def dtype(self):
        return _PRECISIONS[self.precision]

    @property
    def torch_dtype(self):
        return _TORCH[self.precision]

    @classmethod
    def for_inputs(cls, q: np.ndarray, **kw) -> "AttentionConfig":
        return cls(n=q.shape[0], d=q.shape[1], **kw)


@dataclass
class GradBundle:
    """(dq, dk, dv), iterable (oracles.py:41-50)."""

    dq: np.ndarray
    dk: np.ndarray
    dv: np.ndarray

    def __iter__(self):
        return iter((self.dq, self.dk, self.dv))


@dataclass
class KvState:
    """The d x d carried summaries (kernels.py:108-121); ``kv_out``/``dkv_out`` of the ABI."""

    kv: np.ndarray
    dkv: np.ndarray

    @classmethod
    def zeros(cls, d: int, dtype=np.float64) -> "KvState":
        return cls(kv=np.zeros((d, d), dtype=dtype), dkv=np.zeros((d, d), dtype=dtype))

    @property
    def nbytes(self) -> int:
        return self.kv.nbytes + self.dkv.nbytes


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("lightning kernels need a CUDA device (B200); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _prep(arrays, cfg: AttentionConfig | None, names="QKV"):
    """kernels.py:133-150: 2-D equal shapes, cfg consistency, finite inputs."""
    first = None
    for a, name in zip(arrays, names):
        if not isinstance(a, np.ndarray) or a.ndim != 2:
            raise ShapeError(f"{name}: expected a 2-D ndarray")
        if first is None:
            first = a.shape
        elif a.shape != first:
            raise ShapeError(f"{name}: shape {a.shape} != {first}")
    if cfg is None:
        cfg = AttentionConfig(n=first[0], d=first[1])
    elif (cfg.n, cfg.d) != first:
        raise ShapeError(f"config says {cfg.n}x{cfg.d}, inputs are {first[0]}x{first[1]}")
    for a, name in zip(arrays, names):
        if not np.isfinite(a).all():
            raise DomainError(f"{name}: contains NaN or Inf")
    dev = _device()
    tensors = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev).to(cfg.torch_dtype)[None, None]
               for a in arrays]
    return tensors, cfg


def _host(t: torch.Tensor, cfg: AttentionConfig) -> np.ndarray:
    return t[0, 0].to(torch.float64 if cfg.precision == "reference" else torch.float32).cpu().numpy()


def _require_lam_one(cfg: AttentionConfig, who: str) -> None:
    if cfg.lam != 1.0:
        raise DomainError(f"{who} is the undecayed kernel; lam must be 1, got {cfg.lam} (use the decay variant)")


def lightning_forward_decay(q, k, v, cfg: AttentionConfig | None = None) -> np.ndarray:
    (tq, tk, tv), cfg = _prep([q, k, v], cfg)
    o = ops.la_forward(tq, tk, tv, cfg.lam, block=cfg.block)
    out = _host(o, cfg)
    if not np.isfinite(out).all():  # kernels.py:284
        raise DomainError("lightning decay output: contains NaN or Inf")
    return out


def lightning_forward(q, k, v, cfg: AttentionConfig | None = None) -> np.ndarray:
    (tq, tk, tv), cfg = _prep([q, k, v], cfg)
    _require_lam_one(cfg, "lightning_forward")
    return _host(ops.la_forward(tq, tk, tv, 1.0, block=cfg.block), cfg)


def lightning_backward_decay(q, k, v, do, cfg: AttentionConfig | None = None) -> GradBundle:
    (tq, tk, tv, tdo), cfg = _prep([q, k, v, do], cfg, names=["Q", "K", "V", "dO"])
    dq, dk, dv = ops.la_backward(tq, tk, tv, tdo, cfg.lam, block=cfg.block)
    return GradBundle(dq=_host(dq, cfg), dk=_host(dk, cfg), dv=_host(dv, cfg))


def lightning_backward(q, k, v, do, cfg: AttentionConfig | None = None) -> GradBundle:
    (tq, tk, tv, tdo), cfg = _prep([q, k, v, do], cfg, names=["Q", "K", "V", "dO"])
    _require_lam_one(cfg, "lightning_backward")
    dq, dk, dv = ops.la_backward(tq, tk, tv, tdo, 1.0, block=cfg.block)
    return GradBundle(dq=_host(dq, cfg), dk=_host(dk, cfg), dv=_host(dv, cfg))


# ---------------------------------------------------------------------------
# timing and auxiliary-memory accounting (kernels.py:342-471)
# ---------------------------------------------------------------------------


def aux_state_bytes(kind: str, n: int, d: int, block: int, itemsize: int, backward: bool = False) -> int:
    """Device bytes beyond inputs/outputs: the library workspace plus the carried states.

    The workspace holds per-segment summaries; the segment count is capped by
    the SM count, so like the reference's inventory it does not grow with n.
    The "left" / "right" baselines keep the reference's analytic inventory
    (kernels.py:356-359): n x n score + mask, or the d x d summary + one temp.
    """
    if kind not in KERNEL_KINDS:
        raise DomainError(f"unknown kernel kind {kind!r}, expected one of {KERNEL_KINDS}")
    if kind == "left":
        return 2 * n * n * itemsize
    if kind == "right":
        return 2 * d * d * itemsize
    dtype = {8: torch.float64, 4: torch.float32, 2: torch.bfloat16}.get(itemsize)
    if dtype is None:
        raise DomainError(f"itemsize must be 8, 4 or 2, got {itemsize}")
    ws = ops.workspace_bytes((1, 1, n, d), dtype)
    states = (2 if backward else 1) * d * d * max(itemsize, 4)
    return ws + states


@dataclass(frozen=True)
class TimingRecord:
    """One timed kernel invocation (kernels.py:371-391), same CSV schema."""

    kernel: str
    n: int
    d: int
    B: int
    lam: float
    pass_name: str
    median_ns: int
    per_token_ns: float
    aux_bytes: int

    CSV_HEADER = "kernel,n,d,B,lambda,pass,median_ns,per_token_ns,aux_bytes"

    def csv_row(self) -> str:
        return (f"{self.kernel},{self.n},{self.d},{self.B},{self.lam:g},{self.pass_name},"
                f"{self.median_ns},{self.per_token_ns:.3f},{self.aux_bytes}")


def bench_kernel(kind: str, cfg: AttentionConfig, repeats: int, backward: bool = False, seed: int = 0) -> TimingRecord:
    """kernels.py:418-471 on the device: seeded inputs resident in HBM, one warm-up,
    median of ``repeats`` CUDA-event timings of the kernel launch sequence."""
    if repeats < 3:
        raise DomainError(f"repeats must be >= 3, got {repeats}")
    if kind not in KERNEL_KINDS:
        raise DomainError(f"unknown kernel kind {kind!r}, expected one of {KERNEL_KINDS}")
    if kind == "lightning":
        _require_lam_one(cfg, "bench of the undecayed kernel")
    dev = _device()
    rng = np.random.default_rng(seed)
    tdt = cfg.torch_dtype if kind.startswith("lightning") else torch.float64  # left / right: fp64 baselines
    mats = [torch.from_numpy(rng.standard_normal((cfg.n, cfg.d))).to(dev).to(tdt)[None, None]
            for _ in range(4 if backward else 3)]
    lam_dev = ops.decay_tensor(cfg.lam, 1, dev)
    if kind == "left":
        call = (lambda: left_product_backward_device(*mats, cfg.lam)) if backward else \
            (lambda: left_product_forward_device(*mats, cfg.lam))  # noqa: E731
    elif kind == "right":
        call = (lambda: right_product_backward_device(*mats, lam_dev)) if backward else \
            (lambda: right_product_forward_device(*mats, lam_dev))  # noqa: E731
    elif backward:
        call = lambda: ops.la_backward(*mats, None, lam_dev=lam_dev)  # noqa: E731
    else:
        call = lambda: ops.la_forward(*mats, None, lam_dev=lam_dev)  # noqa: E731
    call()
    times = []
    for _ in range(repeats):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        call()
        end.record()
        end.synchronize()
        times.append(int(start.elapsed_time(end) * 1e6))
    med = int(median(times))
    itemsize = torch.empty(0, dtype=tdt).element_size()
    return TimingRecord(kernel=kind, n=cfg.n, d=cfg.d, B=cfg.block, lam=cfg.lam,
                        pass_name="bwd" if backward else "fwd", median_ns=med, per_token_ns=med / cfg.n,
                        aux_bytes=aux_state_bytes(kind, cfg.n, cfg.d, cfg.block, itemsize, backward))


# ---------------------------------------------------------------------------
# the timing harness's baselines on the device (oracles.py:100-162)
# ---------------------------------------------------------------------------


def _decay_mask(n: int, lam: float, like: torch.Tensor) -> torch.Tensor:
    """M[t, s] = lam^(t-s) for t >= s, else 0 (matrixops.py:122-140), built in fp64."""
    t = torch.arange(n, device=like.device)
    diff = (t[:, None] - t[None, :]).to(torch.float64)
    m = torch.where(diff >= 0, torch.pow(torch.tensor(lam, dtype=torch.float64, device=like.device),
                                         diff.clamp(min=0)), torch.zeros((), dtype=torch.float64, device=like.device))
    return m.to(like.dtype)


def left_product_forward_device(q, k, v, lam: float):
    """O = [(Q K^T) * M] V (oracles.py:100-115) with cuBLAS GEMMs; q, k, v [b, h, n, d]."""
    m = _decay_mask(q.shape[-2], lam, q)
    return ((q @ k.transpose(-1, -2)) * m) @ v


def left_product_backward_device(q, k, v, do, lam: float):
    """dV = S^T dO, dS = (dO V^T) * M, dQ = dS K, dK = dS^T Q (oracles.py:164-178)."""
    m = _decay_mask(q.shape[-2], lam, q)
    sc = (q @ k.transpose(-1, -2)) * m
    ds = (do @ v.transpose(-1, -2)) * m
    return ds @ k, ds.transpose(-1, -2) @ q, sc.transpose(-1, -2) @ do


def _recurrent_walk(a, b, c, lam_dev, reverse: bool):
    """out_t = a_t . S_t with S_t = lam S_(t-+1) + b_t c_t^T, one la_decode per position."""
    bsz, h, n, d = a.shape
    st = torch.zeros(bsz, h, d, d, dtype=ops.state_dtype(a.dtype), device=a.device)
    out = torch.empty_like(a)
    for t in (range(n - 1, -1, -1) if reverse else range(n)):
        out[:, :, t] = ops.la_decode(a[:, :, t], b[:, :, t], c[:, :, t], None, st, lam_dev=lam_dev)
    return out


def right_product_forward_device(q, k, v, lam_dev):
    """kv_t = lam kv_(t-1) + k_t v_t^T, o_t = q_t kv_t (oracles.py:118-131)."""
    return _recurrent_walk(q, k, v, lam_dev, reverse=False)


def right_product_backward_device(q, k, v, do, lam_dev):
    """reference_backward's sweeps (oracles.py:134-161): dq_t = do_t kv_t^T (forward walk over
    (v, k)), dk_t = v_t dkv_t^T and dv_t = k_t dkv_t (reverse walks over (do, q) and (q, do))."""
    return (_recurrent_walk(do, v, k, lam_dev, reverse=False), _recurrent_walk(v, do, q, lam_dev, reverse=True),
            _recurrent_walk(k, q, do, lam_dev, reverse=True))
