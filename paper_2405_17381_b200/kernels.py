"""Reference-compatible adapter: the ``linattn.kernels`` call surface on the GPU.

Same names, argument meaning and error behaviour as the reference
(kernels.py:64-471), so its tests and harness can be re-pointed here:

    AttentionConfig(n, d, B=None, lam=1.0, precision="reference")   kernels.py:69-105
    lightning_forward(q, k, v, cfg)          -> ndarray              kernels.py:158-183
    lightning_backward(q, k, v, do, cfg)     -> GradBundle           kernels.py:186-231
    lightning_forward_decay(q, k, v, cfg)    -> ndarray              kernels.py:253-284
    lightning_backward_decay(q, k, v, do, cfg) -> GradBundle         kernels.py:287-334
    KvState, GradBundle, TimingRecord, bench_kernel, aux_state_bytes

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

KERNEL_KINDS = ("lightning", "lightning-decay")

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
    """
    if kind not in KERNEL_KINDS:
        raise DomainError(f"unknown kernel kind {kind!r}, expected one of {KERNEL_KINDS}")
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
    mats = [torch.from_numpy(rng.standard_normal((cfg.n, cfg.d))).to(dev).to(cfg.torch_dtype)[None, None]
            for _ in range(4 if backward else 3)]
    lam_dev = ops.decay_tensor(cfg.lam, 1, dev)
    if backward:
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
    itemsize = torch.empty(0, dtype=cfg.torch_dtype).element_size()
    return TimingRecord(kernel=kind, n=cfg.n, d=cfg.d, B=cfg.block, lam=cfg.lam,
                        pass_name="bwd" if backward else "fwd", median_ns=med, per_token_ns=med / cfg.n,
                        aux_bytes=aux_state_bytes(kind, cfg.n, cfg.d, cfg.block, itemsize, backward))
