"""ctypes binding of the C ABI in ``include/lightning_attn.h``.

The library is built in-tree (``paper_2405_17381_b200/libla_b200.so``, see
``build.py``).  There is deliberately no fallback: if the library is missing
or fails to load, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_void_p
from pathlib import Path

from .errors import DomainError, ShapeError

LIB_PATH = Path(os.environ.get("LA_B200_LIB", Path(__file__).resolve().parent / "libla_b200.so"))

LA_OK, LA_ERR_SHAPE, LA_ERR_DOMAIN, LA_ERR_CUDA, LA_ERR_UNSUPPORTED = range(5)
LA_F32, LA_F64, LA_BF16 = 0, 1, 2
LA_BACKEND_AUTO, LA_BACKEND_SIMT, LA_BACKEND_TCGEN05 = 0, 1, 2
BACKENDS = {"auto": LA_BACKEND_AUTO, "simt": LA_BACKEND_SIMT, "tcgen05": LA_BACKEND_TCGEN05}

# every symbol include/lightning_attn.h declares
EXPORTS = ("la_workspace_bytes", "la_segment_count", "la_fwd", "la_bwd", "la_fwd_ex", "la_bwd_ex", "la_check_decay",
           "la_fwd_state", "la_bwd_state",
           "la_decode", "la_gla_workspace_bytes", "la_gla_prologue", "la_gla_prologue_bwd", "la_gla_epilogue",
           "la_gla_epilogue_bwd", "la_gla_core_fwd", "la_gla_core_workspace_bytes",
           "la_gla_core_bwd", "la_gla_core_bwd_workspace_bytes", "la_gla_gate_rowsq", "la_gla_rowscale", "la_launch_count", "la_last_error", "la_abi_version", "la_build_info")
ABI_VERSION = 4
# la_fwd_ex / la_bwd_ex flags
LA_FLAG_RESUME, LA_FLAG_CHECK_DECAY, LA_FLAG_CHECK_FINITE, LA_FLAG_NO_DQ, LA_FLAG_NO_DKDV = 0x1, 0x2, 0x4, 0x8, 0x10
# la_operand
LA_T_Q, LA_T_K, LA_T_V, LA_T_O, LA_T_DO, LA_T_DQ, LA_T_DK, LA_T_DV = range(8)
LA_ACT_NONE, LA_ACT_SWISH, LA_ACT_ONE_PLUS_ELU = 0, 1, 2
ACTS = {"none": LA_ACT_NONE, "swish": LA_ACT_SWISH, "one_plus_elu": LA_ACT_ONE_PLUS_ELU}


class LaDesc(ctypes.Structure):
    """Mirror of ``la_desc``."""

    _fields_ = [
        ("batch", c_int64),
        ("heads", c_int64),
        ("n", c_int64),
        ("d", c_int64),
        ("block", c_int64),
        ("dtype", c_int32),
        ("backend", c_int32),
        ("stride", c_int64 * 3),
        ("segments", c_int64),
    ]


class LaTensorStrides(ctypes.Structure):
    """Mirror of ``la_tensor_strides``: [la_operand][batch, head, position] element strides."""

    _fields_ = [("s", (c_int64 * 3) * 8)]


class LaGlaDesc(ctypes.Structure):
    """Mirror of ``la_gla_desc``."""

    _fields_ = [
        ("batch", c_int64),
        ("n", c_int64),
        ("heads", c_int64),
        ("d", c_int64),
        ("dtype", ctypes.c_int32),
        ("act", ctypes.c_int32),
        ("offset", c_int64),
        ("eps", c_double),
    ]


class LibraryMissing(RuntimeError):
    """The CUDA library is not built / not loadable; there is no CPU fallback."""


class UnsupportedError(NotImplementedError):
    """LA_ERR_UNSUPPORTED: a valid request this build does not implement."""


class CudaError(RuntimeError):
    """LA_ERR_CUDA: launch or runtime failure inside the library."""


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise LibraryMissing(
            f"{LIB_PATH} not found: build it with `python -m paper_2405_17381_b200.build` "
            "(this package has no CPU fallback)")
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise LibraryMissing(f"failed to load {LIB_PATH}: {exc}") from exc
    P = POINTER(LaDesc)
    lib.la_workspace_bytes.argtypes = [P]
    lib.la_workspace_bytes.restype = c_size_t
    lib.la_segment_count.argtypes = [P]
    lib.la_segment_count.restype = c_int
    lib.la_fwd.argtypes = [P, c_void_p, c_void_p, c_void_p, POINTER(c_double), c_void_p, c_void_p, c_void_p,
                           c_void_p, c_void_p, c_size_t, c_void_p]
    lib.la_fwd.restype = c_int
    lib.la_bwd.argtypes = [P, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_double), c_void_p, c_void_p,
                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
    lib.la_bwd.restype = c_int
    S = POINTER(LaTensorStrides)
    lib.la_fwd_ex.argtypes = [P, S, ctypes.c_uint32, c_void_p, c_void_p, c_void_p, POINTER(c_double), c_void_p,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
    lib.la_fwd_ex.restype = c_int
    lib.la_bwd_ex.argtypes = [P, S, ctypes.c_uint32, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_double),
                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_size_t, c_void_p]
    lib.la_bwd_ex.restype = c_int
    lib.la_check_decay.argtypes = [POINTER(c_double), c_int64]
    lib.la_check_decay.restype = c_int
    lib.la_fwd_state.argtypes = [P, c_void_p, c_void_p, POINTER(c_double), c_void_p, c_void_p, c_size_t, c_void_p]
    lib.la_fwd_state.restype = c_int
    lib.la_bwd_state.argtypes = [P, c_void_p, c_void_p, POINTER(c_double), c_void_p, c_void_p, c_size_t, c_void_p]
    lib.la_bwd_state.restype = c_int
    lib.la_decode.argtypes = [P, c_void_p, c_void_p, c_void_p, POINTER(c_double), c_void_p, c_void_p, c_void_p]
    lib.la_decode.restype = c_int
    G = POINTER(LaGlaDesc)
    lib.la_gla_workspace_bytes.argtypes = [G]
    lib.la_gla_workspace_bytes.restype = c_size_t
    lib.la_gla_prologue.argtypes = [G, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.la_gla_prologue.restype = c_int
    lib.la_gla_prologue_bwd.argtypes = [G, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_size_t, c_void_p]
    lib.la_gla_prologue_bwd.restype = c_int
    lib.la_gla_epilogue.argtypes = [G, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.la_gla_epilogue.restype = c_int
    lib.la_gla_epilogue_bwd.argtypes = [G, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.la_gla_epilogue_bwd.restype = c_int
    # the fused GLA core entry points (ABI 4) are bound when present, so A/B experiments can load an older build;
    # calling one that is missing raises AttributeError (build() checks every export of the shipped library)
    if hasattr(lib, "la_gla_core_fwd"):
        lib.la_gla_core_fwd.argtypes = [G, c_void_p, c_void_p, c_void_p, POINTER(c_double), c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
        lib.la_gla_core_fwd.restype = c_int
        lib.la_gla_core_workspace_bytes.argtypes = [G]
        lib.la_gla_core_workspace_bytes.restype = c_size_t
    if hasattr(lib, "la_gla_core_bwd"):
        lib.la_gla_core_bwd.argtypes = [G, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        POINTER(c_double), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_size_t, c_void_p]
        lib.la_gla_core_bwd.restype = c_int
        lib.la_gla_core_bwd_workspace_bytes.argtypes = [G]
        lib.la_gla_core_bwd_workspace_bytes.restype = c_size_t
    lib.la_gla_gate_rowsq.argtypes = [G, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]
    lib.la_gla_gate_rowsq.restype = c_int
    lib.la_gla_rowscale.argtypes = [c_int, c_int64, c_int64, c_double, c_void_p, c_void_p, c_void_p]
    lib.la_gla_rowscale.restype = c_int
    lib.la_launch_count.argtypes = [P, c_int]
    lib.la_launch_count.restype = c_int
    lib.la_last_error.argtypes = []
    lib.la_last_error.restype = c_char_p
    lib.la_abi_version.argtypes = []
    lib.la_abi_version.restype = c_int
    lib.la_build_info.argtypes = []
    lib.la_build_info.restype = c_char_p
    _lib = lib
    return lib


def check(status: int) -> None:
    """Map an la_status onto the reference's exception classes (matrixops.py:28-33)."""
    if status == LA_OK:
        return
    msg = load().la_last_error().decode(errors="replace")
    if status == LA_ERR_SHAPE:
        raise ShapeError(msg)
    if status == LA_ERR_DOMAIN:
        raise DomainError(msg)
    if status == LA_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise CudaError(msg)
