"""B200-native Lightning Attention (arXiv 2405.17381): the reference ``linattn``
hot path -- tiled causal linear attention with per-head decay, forward and
backward -- as hand-written sm_100a CUDA behind a C ABI.

Public surface:
  * ``LightningAttention`` / ``lightning_attention``: batched autograd op on
    torch CUDA tensors ([batch, heads, n, d] or [batch, n, heads, d]).
  * ``ops``: explicit forward / backward / state entry points with kv_in /
    kv_out and dkv_in / dkv_out for segment chaining.
  * reference-compatible names (``AttentionConfig``, ``lightning_forward_decay``,
    ``lightning_backward_decay``, ``lightning_forward``, ``lightning_backward``,
    ``GradBundle``, ``KvState``, ``ShapeError``, ``DomainError``, ...).
  * ``sp``: sequence parallelism over NCCL (state passing between ranks).
"""

from .errors import DomainError, ShapeError
from .positional import DecaySchedule, decay_rate

__version__ = "0.1.0"

_LAZY = {
    "LightningAttention": ("attention", "LightningAttention"),
    "lightning_attention": ("attention", "lightning_attention"),
    "AttentionConfig": ("kernels", "AttentionConfig"),
    "GradBundle": ("kernels", "GradBundle"),
    "KvState": ("kernels", "KvState"),
    "TimingRecord": ("kernels", "TimingRecord"),
    "KERNEL_KINDS": ("kernels", "KERNEL_KINDS"),
    "aux_state_bytes": ("kernels", "aux_state_bytes"),
    "bench_kernel": ("kernels", "bench_kernel"),
    "lightning_forward": ("kernels", "lightning_forward"),
    "lightning_backward": ("kernels", "lightning_backward"),
    "lightning_forward_decay": ("kernels", "lightning_forward_decay"),
    "lightning_backward_decay": ("kernels", "lightning_backward_decay"),
    "BenchGrid": ("records", "BenchGrid"),
    "run_bench": ("records", "run_bench"),
    "write_csv": ("records", "write_csv"),
    "read_csv": ("records", "read_csv"),
}


def __getattr__(name):  # torch is imported lazily so `import` stays cheap
    if name in _LAZY:
        import importlib

        mod, attr = _LAZY[name]
        return getattr(importlib.import_module(f"{__name__}.{mod}"), attr)
    raise AttributeError(name)


__all__ = ["DomainError", "ShapeError", "DecaySchedule", "decay_rate", *_LAZY]
