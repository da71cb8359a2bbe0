"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and validates descriptors exactly like the reference's
AttentionConfig/_prep (no device work happens on these paths)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2405_17381_b200 import _lib
from paper_2405_17381_b200.errors import DomainError, ShapeError

HEADER = Path(__file__).resolve().parent.parent / "include" / "lightning_attn.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"LA_API\s+[\w\s\*]+?\b(la_\w+)\s*\(", text)))


def test_header_declares_what_binding_expects():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.la_abi_version() == _lib.ABI_VERSION == 4
    assert b"sm_100a" in lib.la_build_info()


def _desc(**kw):
    d = _lib.LaDesc()
    d.batch, d.heads, d.n, d.d = kw.get("batch", 1), kw.get("heads", 2), kw.get("n", 64), kw.get("d", 16)
    d.block = kw.get("block", 0)
    d.dtype = kw.get("dtype", _lib.LA_F32)
    d.backend = kw.get("backend", _lib.LA_BACKEND_AUTO)
    s = kw.get("stride", (d.heads * d.n * d.d, d.n * d.d, d.d))
    for i in range(3):
        d.stride[i] = s[i]
    d.segments = kw.get("segments", 0)
    return d


def _fwd(desc):
    lib = _lib.load()
    dummy = ctypes.c_void_p(16)
    lam = ctypes.cast(ctypes.c_void_p(16), ctypes.POINTER(ctypes.c_double))
    return lib.la_fwd(ctypes.byref(desc), dummy, dummy, dummy, lam, None, dummy, None, None, None, 0, None)


@pytest.mark.parametrize("kw,code", [
    (dict(n=0), _lib.LA_ERR_DOMAIN),            # kernels.py:85-86
    (dict(d=0), _lib.LA_ERR_DOMAIN),
    (dict(block=-1), _lib.LA_ERR_DOMAIN),       # kernels.py:90-91
    (dict(dtype=7), _lib.LA_ERR_DOMAIN),        # kernels.py:88-89 (precision)
    (dict(batch=0), _lib.LA_ERR_SHAPE),
    (dict(stride=(0, 0, 3)), _lib.LA_ERR_SHAPE),
    (dict(d=256), _lib.LA_ERR_UNSUPPORTED),
    (dict(segments=70000), _lib.LA_ERR_UNSUPPORTED),      # beyond the workspace's segment bound
    (dict(n=2 ** 31), _lib.LA_ERR_UNSUPPORTED),           # int positions
    (dict(segments=-1), _lib.LA_ERR_DOMAIN),
    (dict(dtype=_lib.LA_F64, backend=_lib.LA_BACKEND_TCGEN05), _lib.LA_ERR_UNSUPPORTED),
])
def test_descriptor_validation(kw, code):
    assert _fwd(_desc(**kw)) == code
    assert _lib.load().la_last_error()


def test_status_maps_to_reference_exceptions():
    with pytest.raises(DomainError):
        _lib.check(_fwd(_desc(n=0)))
    with pytest.raises(ShapeError):
        _lib.check(_fwd(_desc(batch=0)))
    with pytest.raises(_lib.UnsupportedError):
        _lib.check(_fwd(_desc(d=512)))


def test_workspace_is_bounded_in_n():
    lib = _lib.load()
    sizes = set()
    for n in (1 << 14, 1 << 17, 1 << 20):
        sizes.add(lib.la_workspace_bytes(ctypes.byref(_desc(n=n, d=128, heads=16, dtype=_lib.LA_BF16))))
    assert len(sizes) == 1, sizes
    assert lib.la_workspace_bytes(ctypes.byref(_desc(n=0))) == 0


def test_segment_count_and_launches_follow_the_plan():
    lib = _lib.load()
    short = _desc(batch=64, heads=16, n=1024, d=128, dtype=_lib.LA_BF16)
    long_ = _desc(batch=1, heads=16, n=1 << 17, d=128, dtype=_lib.LA_BF16)
    assert lib.la_segment_count(ctypes.byref(short)) == 1
    # tcgen05 backend: bwd = dq pass + one fused dk/dv sweep
    assert lib.la_launch_count(ctypes.byref(short), 0) == 1 and lib.la_launch_count(ctypes.byref(short), 1) == 2
    assert lib.la_segment_count(ctypes.byref(long_)) > 1
    assert [lib.la_launch_count(ctypes.byref(long_), w) for w in (0, 1, 2)] == [3, 6, 4]
    assert lib.la_segment_count(ctypes.byref(_desc(n=0))) == -1


def test_decay_tensor_is_validated_once_and_cached():
    """Host decays are validated and copied once per (values, device); later calls reuse the tensor
    (no per-call host-to-device copy in the autograd ops), invalid values still raise every time."""
    import torch
    from paper_2405_17381_b200 import ops
    from paper_2405_17381_b200.errors import DomainError, ShapeError
    a = ops.decay_tensor([0.9, 0.5], 2, "cpu")
    assert a is ops.decay_tensor([0.9, 0.5], 2, torch.device("cpu"))
    assert a is not ops.decay_tensor([0.9, 0.6], 2, "cpu")
    assert ops.decay_tensor(0.7, 3, "cpu").tolist() == [0.7, 0.7, 0.7]
    for bad in ([1.5, 0.5], [0.0, 0.5]):
        with pytest.raises(DomainError):
            ops.decay_tensor(bad, 2, "cpu")
    with pytest.raises(ShapeError):
        ops.decay_tensor([0.9, 0.5, 0.4], 2, "cpu")


def test_check_decay_host_entry_matches_reference_check_decay():
    """la_check_decay: the reference's check_decay (matrixops.py:72-77) on a host array."""
    lib = _lib.load()
    arr = lambda *v: (ctypes.c_double * len(v))(*v)  # noqa: E731
    assert lib.la_check_decay(arr(1.0, 0.5, 5.5e-4), 3) == _lib.LA_OK
    for bad in (1.5, 0.0, -0.2, float("nan"), float("inf")):
        assert lib.la_check_decay(arr(0.9, bad), 2) == _lib.LA_ERR_DOMAIN
        assert b"(0, 1]" in lib.la_last_error()
    assert lib.la_check_decay(None, 2) == _lib.LA_ERR_SHAPE


def _fwd_ex(desc, strides=None, flags=0):
    lib = _lib.load()
    dummy = ctypes.c_void_p(16)
    lam = ctypes.cast(ctypes.c_void_p(16), ctypes.POINTER(ctypes.c_double))
    sp = ctypes.byref(strides) if strides is not None else None
    return lib.la_fwd_ex(ctypes.byref(desc), sp, flags, dummy, dummy, dummy, lam, None, dummy, None, None, None, 0,
                         None)


def test_extended_entry_validation():
    """la_fwd_ex / la_bwd_ex reject unknown or misplaced flags and bad per-operand strides before any
    device work."""
    lib = _lib.load()
    assert _fwd_ex(_desc(), flags=0x400) == _lib.LA_ERR_DOMAIN
    assert _fwd_ex(_desc(), flags=_lib.LA_FLAG_NO_DQ) == _lib.LA_ERR_DOMAIN  # backward-only flag
    st = _lib.LaTensorStrides()
    for i in range(8):
        st.s[i][0], st.s[i][1], st.s[i][2] = 2 * 64 * 16, 64 * 16, 16
    st.s[_lib.LA_T_V][2] = 8  # position stride < d
    assert _fwd_ex(_desc(), st) == _lib.LA_ERR_SHAPE
    assert b"operand 2" in lib.la_last_error()
    st.s[_lib.LA_T_V][2] = 16
    st.s[_lib.LA_T_K][0] = -1
    assert _fwd_ex(_desc(), st) == _lib.LA_ERR_SHAPE
    dummy = ctypes.c_void_p(16)
    lam = ctypes.cast(ctypes.c_void_p(16), ctypes.POINTER(ctypes.c_double))
    # NO_DKDV without dq, RESUME on a split problem without the forward's segment states
    long_ = _desc(batch=1, heads=16, n=1 << 17, d=128, dtype=_lib.LA_BF16)
    ws = ctypes.create_string_buffer(lib.la_workspace_bytes(ctypes.byref(long_)) + 16)
    wsp = ctypes.c_void_p((ctypes.addressof(ws) + 15) // 16 * 16)
    rc = lib.la_bwd_ex(ctypes.byref(long_), None, _lib.LA_FLAG_NO_DKDV, dummy, dummy, dummy, dummy, lam, None, None,
                       None, None, None, None, None, wsp, len(ws) - 16, None)
    assert rc == _lib.LA_ERR_SHAPE
    rc = lib.la_bwd_ex(ctypes.byref(long_), None, _lib.LA_FLAG_RESUME, dummy, dummy, dummy, dummy, lam, None, None,
                       None, dummy, dummy, dummy, None, wsp, len(ws) - 16, None)
    assert rc == _lib.LA_ERR_SHAPE and b"fwd_seg_states" in lib.la_last_error()


def test_workspace_covers_every_backend_plan():
    """An _ex call whose operand strides rule out TMA runs the SIMT plan: la_workspace_bytes covers it."""
    lib = _lib.load()
    for n in (1 << 12, 1 << 16):
        tc = _desc(batch=1, heads=4, n=n, d=128, dtype=_lib.LA_BF16)
        simt = _desc(batch=1, heads=4, n=n, d=128, dtype=_lib.LA_BF16, backend=_lib.LA_BACKEND_SIMT)
        assert lib.la_workspace_bytes(ctypes.byref(tc)) >= lib.la_workspace_bytes(ctypes.byref(simt))


def _gla_desc(**kw):
    d = _lib.LaGlaDesc()
    d.batch, d.n, d.heads, d.d = kw.get("batch", 2), kw.get("n", 300), kw.get("heads", 16), kw.get("d", 128)
    d.dtype = kw.get("dtype", _lib.LA_BF16)
    d.act = kw.get("act", _lib.LA_ACT_SWISH)
    d.offset = kw.get("offset", 0)
    d.eps = 1e-8
    return d


def test_gla_core_entry_validation():
    """la_gla_core_fwd / la_gla_core_bwd (ABI 4) reject bad descriptors, missing operands, lone q_out / k_out,
    misaligned rows and non-tensor-core shapes before any device work; their workspace sizes follow the
    attention plan (0 when sequences are not split)."""
    lib = _lib.load()
    d16 = ctypes.c_void_p(16)
    lam = ctypes.cast(ctypes.c_void_p(16), ctypes.POINTER(ctypes.c_double))

    def fwd(desc, qp=d16, q_out=None, k_out=None):
        return lib.la_gla_core_fwd(ctypes.byref(desc), qp, d16, d16, lam, None, None, d16, q_out, k_out, None, None,
                                   0, None)

    def bwd(desc, dqp=d16):
        return lib.la_gla_core_bwd(ctypes.byref(desc), d16, d16, d16, d16, d16, d16, lam, None, None, None, dqp, d16,
                                   d16, None, None, 0, None)

    assert fwd(_gla_desc(n=0)) == _lib.LA_ERR_DOMAIN
    assert fwd(_gla_desc(act=9)) == _lib.LA_ERR_DOMAIN
    assert fwd(_gla_desc(offset=-1)) == _lib.LA_ERR_DOMAIN
    assert fwd(_gla_desc(), qp=None) == _lib.LA_ERR_SHAPE
    assert fwd(_gla_desc(), q_out=d16) == _lib.LA_ERR_SHAPE and b"together" in lib.la_last_error()
    assert fwd(_gla_desc(), qp=ctypes.c_void_p(24)) == _lib.LA_ERR_SHAPE  # rows must be 16-byte aligned
    assert fwd(_gla_desc(dtype=_lib.LA_F32)) == _lib.LA_ERR_UNSUPPORTED
    assert fwd(_gla_desc(d=64, heads=32)) == _lib.LA_ERR_UNSUPPORTED
    assert bwd(_gla_desc(), dqp=None) == _lib.LA_ERR_SHAPE
    assert bwd(_gla_desc(dtype=_lib.LA_F64)) == _lib.LA_ERR_UNSUPPORTED
    full = _gla_desc(batch=8, n=8192)           # batch x heads = 128: one unsplit wave
    split = _gla_desc(batch=1, n=1 << 16)       # 16 sequences: split into segments
    assert lib.la_gla_core_workspace_bytes(ctypes.byref(full)) == 0
    assert lib.la_gla_core_workspace_bytes(ctypes.byref(split)) > 0
    assert lib.la_gla_core_bwd_workspace_bytes(ctypes.byref(split)) >= lib.la_gla_core_workspace_bytes(
        ctypes.byref(split))
    assert lib.la_gla_core_workspace_bytes(ctypes.byref(_gla_desc(dtype=_lib.LA_F32))) == 0


def test_fp32_tensor_core_backend_selection():
    """fp32 at d = 128 with 16-byte strides is served by the tcgen05 split pass (its own plan: one wave of
    segments for a long sequence, bounded workspace); head dims that are not a multiple of 32 cannot be forced
    onto the tensor cores."""
    lib = _lib.load()
    long32 = _desc(batch=1, heads=16, n=1 << 17, d=128, dtype=_lib.LA_F32, backend=_lib.LA_BACKEND_TCGEN05)
    assert lib.la_segment_count(ctypes.byref(long32)) == 148 // 16
    sizes = {lib.la_workspace_bytes(ctypes.byref(_desc(batch=1, heads=16, n=n, d=128, dtype=_lib.LA_F32)))
             for n in (1 << 14, 1 << 17, 1 << 20)}
    assert len(sizes) == 1 and sizes.pop() > 0
    # backward on the split pass: three passes (no fused dK/dV sweep in fp32)
    assert lib.la_launch_count(ctypes.byref(_desc(batch=64, heads=16, n=1024, d=128, dtype=_lib.LA_F32)), 1) == 3
    # head dims below 128 run on zero-padded features when they are a multiple of 32 (both dtypes)
    for dt in (_lib.LA_F32, _lib.LA_BF16):
        for d in (32, 64, 96):
            assert lib.la_segment_count(ctypes.byref(_desc(d=d, dtype=dt, backend=_lib.LA_BACKEND_TCGEN05))) >= 1
        for d in (16, 48):
            assert _fwd(_desc(d=d, dtype=dt, backend=_lib.LA_BACKEND_TCGEN05)) == _lib.LA_ERR_UNSUPPORTED
    assert _fwd(_desc(d=128, dtype=_lib.LA_F32, backend=_lib.LA_BACKEND_TCGEN05, stride=(2 * 64 * 130, 64 * 130, 130))) \
        == _lib.LA_ERR_UNSUPPORTED  # a position stride of 130 floats is not 16-byte aligned
