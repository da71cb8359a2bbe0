"""ABI 3 on the GPU: la_fwd_ex / la_bwd_ex per-operand strides, the RESUME and NO_DQ / NO_DKDV flags,
the debug checks (CHECK_DECAY / CHECK_FINITE -> DomainError, as the reference's check_decay and
ensure_finite, matrixops.py:66-77), and the NaN poisoning of an invalid decay that reaches the kernels
through the raw ABI.

Tolerances: bf16 operands with fp32 accumulation <= 2e-2 per-entry relative (positive inputs) against
the oracle; fp32 <= 1e-4; an entry point and its decomposition (resume, parts) must agree bitwise
where they run the same kernels on the same data, else within the dtype's bar.
"""

import ctypes

import numpy as np
import pytest

from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2405_17381_b200 import _lib, ops  # noqa: E402
from paper_2405_17381_b200.errors import DomainError  # noqa: E402

DEV = torch.device("cuda", 0)
TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def host(t):
    return t.detach().to(torch.float64).cpu().numpy()


def _pos(shape, seed, dtype):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return (torch.rand(*shape, device=DEV, generator=g) * 0.95 + 0.05).to(dtype)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_mixed_layouts_need_no_copy(dtype):
    """q, k, v as views into one fused [b, n, 3, h, d] projection (model-native, strided) and dO
    transposed: each operand keeps its own strides -- no copy -- and the result equals the contiguous
    call."""
    b, h, n, d = 2, 4, 700, 128
    lams = [0.999, 0.9, 0.5, 1.0]
    qkv = _pos((b, n, 3, h, d), 11, dtype)
    q, k, v = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]           # [b, n, h, d] views, position stride 3 h d
    do = _pos((b, h, n, d), 12, dtype).transpose(1, 2)             # [b, n, h, d] view of a bhnd tensor
    got_o = ops.la_forward(q, k, v, lams, layout="bnhd")
    got = ops.la_backward(q, k, v, do, lams, layout="bnhd")
    qc, kc, vc, dc = (t.contiguous() for t in (q, k, v, do))
    (qq, kk, vv, _), _ = ops._prep([q, k, v, do], ["Q", "K", "V", "dO"], "bnhd")
    assert qq.data_ptr() == q.data_ptr() and vv.data_ptr() == v.data_ptr()  # passed as is
    want_o = ops.la_forward(qc, kc, vc, lams, layout="bnhd")
    want = ops.la_backward(qc, kc, vc, dc, lams, layout="bnhd")
    assert torch.equal(got_o, want_o)
    for a, w in zip(got, want):
        assert torch.equal(a, w)
    ro, _ = orc.batched_forward(*(host(t.transpose(1, 2)) for t in (q, k, v)), lams)
    assert orc.max_rel_error(host(got_o.transpose(1, 2)), ro) <= TOL[dtype]


@pytest.mark.parametrize("n", [1000, 40000])
def test_resume_equals_plain_forward_and_backward(n):
    """la_fwd_state + la_fwd_ex(RESUME) == la_fwd, la_bwd_state + la_bwd_ex(RESUME, dkdv) == la_bwd's sweep 2,
    bitwise (the same summaries, scans and passes)."""
    b, h, d = 1, 3, 128
    lams = [0.9999, 0.99, 0.4]
    q, k, v, do = (_pos((b, h, n, d), 20 + i, torch.bfloat16) for i in range(4))
    kv_in = torch.rand(b, h, d, d, device=DEV) * 0.01
    ws = ops.new_workspace((b, h, n, d))
    delta = ops.la_forward_state(k, v, lams, workspace=ws)
    (o_r, kv_r), seg_r = ops.la_forward(q, k, v, lams, kv_in=kv_in, want_state=True, want_seg_states=True,
                                        workspace=ws, resume=True)
    (o, kv), seg = ops.la_forward(q, k, v, lams, kv_in=kv_in, want_state=True, want_seg_states=True)
    assert torch.equal(o_r, o) and torch.equal(kv_r, kv)
    assert (seg is None and seg_r is None) or torch.equal(seg_r, seg)
    _, kv0 = ops.la_forward(q, k, v, lams, want_state=True)
    # the summary is F(n) with kv_in = 0 (computed by the summary kernel, bf16 B~ in 64-row chunks)
    assert orc.max_rel_error(host(delta), host(kv0)) <= TOL[torch.bfloat16]
    ws2 = ops.new_workspace((b, h, n, d))
    ops.la_backward_state(q, do, lams, workspace=ws2)
    dkv_in = torch.rand(b, h, d, d, device=DEV) * 0.01
    _, dk_r, dv_r, dkv_r = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, dkv_in=dkv_in, parts="dkdv",
                                           want_state=True, workspace=ws2, resume=True)
    dq_p, _, _ = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, parts="dq", fwd_seg_states=seg)
    dq, dk, dv, dkv = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, dkv_in=dkv_in, want_state=True,
                                      fwd_seg_states=seg)
    assert torch.equal(dk_r, dk) and torch.equal(dv_r, dv) and torch.equal(dkv_r, dkv) and torch.equal(dq_p, dq)


def test_parts_split_matches_full_backward_simt():
    """NO_DQ / NO_DKDV on the SIMT (fp32) path, split sequence."""
    b, h, n, d = 1, 2, 3000, 64
    lams = [0.995, 0.7]
    q, k, v, do = (_pos((b, h, n, d), 30 + i, torch.float32) for i in range(4))
    dq, dk, dv = ops.la_backward(q, k, v, do, lams)
    dq1, n1, n2 = ops.la_backward(q, k, v, do, lams, parts="dq")
    n3, dk1, dv1 = ops.la_backward(q, k, v, do, lams, parts="dkdv")
    assert n1 is None and n2 is None and n3 is None
    for a, w in ((dq1, dq), (dk1, dk), (dv1, dv)):
        assert torch.equal(a, w)


def test_check_flags_raise_the_reference_domain_errors():
    q = _pos((1, 2, 64, 16), 40, torch.float32)
    bad = q.clone()
    bad[0, 1, 7, 3] = float("nan")
    with pytest.raises(DomainError, match="K: contains NaN or Inf"):
        ops.la_forward(q, bad, q, [0.5, 0.9], check=True)
    with pytest.raises(DomainError, match="dO: contains NaN or Inf"):
        ops.la_backward(q, q, q, bad, [0.5, 0.9], check=True)
    ops.la_forward(q, q, q, [0.5, 0.9], check=True)  # clean inputs pass
    # an invalid decay on the device (built around decay_tensor's validation) -> LA_ERR_DOMAIN
    lam_bad = torch.tensor([0.5, 1.5], dtype=torch.float64, device=DEV)
    with pytest.raises(DomainError, match=r"\(0, 1\]"):
        ops.la_forward(q, q, q, None, lam_dev=lam_bad, check=True)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
def test_invalid_decay_through_the_raw_abi_poisons_outputs(dtype):
    """Without the debug flag the kernels read lam through load_decay: lam outside (0, 1] or NaN turns the
    outputs into NaN (never finite garbage), on every backend, segmented or not."""
    d = 128 if dtype == torch.bfloat16 else 32
    for n in (300, 20000):
        q, k, v, do = (_pos((1, 2, n, d), 50 + i, dtype) for i in range(4))
        for badval in (1.5, 0.0, -0.3, float("nan")):
            lam_bad = torch.tensor([0.9, badval], dtype=torch.float64, device=DEV)
            o = ops.la_forward(q, k, v, None, lam_dev=lam_bad)
            dq, dk, dv = ops.la_backward(q, k, v, do, None, lam_dev=lam_bad)
            for t in (o, dq, dk, dv):
                assert torch.isnan(t[:, 1].float()).all(), (n, badval)
                assert torch.isfinite(t[:, 0].float()).all()


def test_check_decay_entry_on_host_values():
    lib = _lib.load()
    arr = (ctypes.c_double * 2)(0.5, 2.0)
    assert lib.la_check_decay(arr, 2) == _lib.LA_ERR_DOMAIN


def test_lam_dev_is_validated_before_the_kernels_read_it():
    """a host tensor, a float32 tensor or the wrong length must not reach the kernels."""
    from paper_2405_17381_b200.errors import ShapeError
    q = _pos((1, 2, 64, 16), 60, torch.float32)
    for lam_dev in (torch.tensor([0.5, 0.9], dtype=torch.float64),
                    torch.tensor([0.5, 0.9], dtype=torch.float32, device=DEV),
                    torch.tensor([0.5], dtype=torch.float64, device=DEV)):
        with pytest.raises(ShapeError):
            ops.la_forward(q, q, q, None, lam_dev=lam_dev)
