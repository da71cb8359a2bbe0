"""Head dims below 128 on the tensor-core backend (la_tc.cu, la_tc_bwd.cu, la_summary.cu, la_tc32.cu).

The tcgen05 kernels are built for d = 128 tiles; a head dim d < 128 (a multiple of 32) runs them on
zero-padded features: the TMA boxes past d read zeros (out-of-bounds fill), TMA stores past d are
clipped, and the carried states are d x d (rows / columns >= d are neither read nor written).  The
zero features contribute exact zeros to every product, so the result is the d-dim attention.

BASELINE.json configs[0] (B = 1, H = 4, n = 1024, d = 64, fp32) is such a case: it now routes to the
fp32 split pass by default.  Bars: fp32 <= 1e-4 relative (positive inputs) / 1e-5 scaled (normal
inputs), bf16 operands <= 2e-2 relative -- as test_gpu_parity.py / test_gpu_tc32.py.  The oracle is
the fp64 restatement of kernels.py:253-334 (pinned by tests/test_oracle.py) on the device's operands.
"""

import numpy as np
import pytest

from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2405_17381_b200 import lightning_attention, ops  # noqa: E402

DEV = torch.device("cuda", 0)
TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}
DTYPES = [torch.float32, torch.bfloat16]
IDS = ["f32", "bf16"]
LAMS3 = [1.0, 0.99, 0.5]


def _inputs(shape, seed, dist="pos", count=4):
    rng = np.random.default_rng(seed)
    if dist == "pos":
        return [rng.uniform(0.05, 1.0, shape) for _ in range(count)]
    return [rng.standard_normal(shape) for _ in range(count)]


def _dev(a, dtype):
    return torch.tensor(a, dtype=torch.float32, device=DEV).to(dtype)


def _host(t):
    return t.detach().double().cpu().numpy()


def _check(got, ref, dtype, what, dist="pos"):
    if dist == "pos":
        err, tol = orc.max_rel_error(_host(got), ref), TOL[dtype]
    else:
        err, tol = orc.max_scaled_error(_host(got), ref), 1e-5
    assert err <= tol, f"{what}: {err:.3e} > {tol:g}"


def _run(dtype, b, h, n, d, lams, seed, *, segments=0, layout="bhnd", dist="pos", backend="tcgen05"):
    q, k, v, do = _inputs((b, h, n, d), seed, dist)
    tq, tk, tv, tdo = (_dev(a, dtype) for a in (q, k, v, do))
    if layout == "bnhd":
        tq, tk, tv, tdo = (t.transpose(1, 2).contiguous().transpose(1, 2) for t in (tq, tk, tv, tdo))
    o = ops.la_forward(tq, tk, tv, lams, backend=backend, segments=segments)
    dq, dk, dv = ops.la_backward(tq, tk, tv, tdo, lams, backend=backend, segments=segments)
    qq, kk, vv, dd = (_host(t) for t in (tq, tk, tv, tdo))
    ro, _ = orc.batched_forward(qq, kk, vv, lams)
    (rdq, rdk, rdv), _ = orc.batched_backward(qq, kk, vv, dd, lams)
    for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        assert got.shape == (b, h, n, d)
        _check(got, ref, dtype, f"{name} d={d} n={n} seg={segments}", dist)


@pytest.mark.parametrize("dtype", DTYPES, ids=IDS)
@pytest.mark.parametrize("d", [32, 64, 96])
@pytest.mark.parametrize("n", [1, 129, 700])
def test_small_d_ragged(dtype, d, n):
    _run(dtype, 2, 3, n, d, LAMS3, seed=d + n)


@pytest.mark.parametrize("dtype", DTYPES, ids=IDS)
@pytest.mark.parametrize("segments", [2, 5])
def test_small_d_forced_segments(dtype, segments):
    """Segmented passes: the summaries export d x d deltas, the scan chains them, the main pass reads them."""
    _run(dtype, 1, 3, 1500, 64, LAMS3, seed=7, segments=segments)
    _run(dtype, 1, 3, 1500, 96, [0.5, 0.05, 5.5e-4], seed=8, segments=segments)


@pytest.mark.parametrize("dtype", DTYPES, ids=IDS)
def test_small_d_model_layout_and_normal_inputs(dtype):
    _run(dtype, 2, 3, 400, 64, LAMS3, seed=9, layout="bnhd")
    if dtype == torch.float32:
        _run(dtype, 2, 3, 500, 64, LAMS3, seed=10, dist="normal")


@pytest.mark.parametrize("dtype", DTYPES, ids=IDS)
@pytest.mark.parametrize("d", [32, 64])
def test_small_d_state_chaining(dtype, d):
    """kv_in / kv_out and dkv_in / dkv_out at d x d: the states match the oracle's."""
    b, h, n = 1, 2, 900
    lams = [0.999, 0.95]
    q, k, v, do = _inputs((b, h, n, d), 31 + d)
    kv0, dkv0 = (np.random.default_rng(32 + d + s).uniform(0.0, 0.5, (b, h, d, d)) for s in range(2))
    tq, tk, tv, tdo = (_dev(a, dtype) for a in (q, k, v, do))
    tkv0, tdkv0 = (_dev(a, torch.float32) for a in (kv0, dkv0))
    o, kv = ops.la_forward(tq, tk, tv, lams, kv_in=tkv0, want_state=True, backend="tcgen05")
    dq, dk, dv, dkv = ops.la_backward(tq, tk, tv, tdo, lams, kv_in=tkv0, dkv_in=tdkv0, want_state=True,
                                      backend="tcgen05")
    assert kv.shape == (b, h, d, d) and dkv.shape == (b, h, d, d)
    qq, kk, vv, dd = (_host(t) for t in (tq, tk, tv, tdo))
    ro, rkv = orc.batched_forward(qq, kk, vv, lams, kv_in=_host(tkv0))
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, lams, kv_in=_host(tkv0), dkv_in=_host(tdkv0))
    for name, got, ref in (("o", o, ro), ("kv", kv, rkv), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv),
                           ("dkv", dkv, rdkv)):
        _check(got, ref, dtype, f"{name} d={d}")


@pytest.mark.parametrize("dtype", DTYPES, ids=IDS)
def test_small_d_matches_simt_backend(dtype):
    """The tensor-core and SIMT backends agree at d = 64 (both meet the bar against the oracle)."""
    q, k, v, do = (_dev(a, dtype) for a in _inputs((1, 4, 777, 64), 21))
    lams = [1.0, 0.99, 0.9, 0.3]
    o_tc = ops.la_forward(q, k, v, lams, backend="tcgen05")
    o_si = ops.la_forward(q, k, v, lams, backend="simt")
    g_tc = ops.la_backward(q, k, v, do, lams, backend="tcgen05")
    g_si = ops.la_backward(q, k, v, do, lams, backend="simt")
    assert orc.max_rel_error(_host(o_tc), _host(o_si)) <= 2 * TOL[dtype]
    for a, b_ in zip(g_tc, g_si):
        assert orc.max_rel_error(_host(a), _host(b_)) <= 2 * TOL[dtype]


def test_config0_default_route_is_tensor_cores():
    """BASELINE.json configs[0] (B = 1, H = 4, n = 1024, d = 64, B_blk = 64, fp32, per-head decay) through
    the autograd op with the default backend: served by the fp32 split pass, parity with the oracle."""
    b, h, n, d = 1, 4, 1024, 64
    lams = [orc.decay_rate(j + 1, 1, h, h) for j in range(h)]
    q, k, v, do = _inputs((b, h, n, d), 41)
    tq, tk, tv = (_dev(a, torch.float32).requires_grad_(True) for a in (q, k, v))
    o = lightning_attention(tq, tk, tv, lams)
    o.backward(_dev(do, torch.float32))
    qq, kk, vv = (_host(t) for t in (tq, tk, tv))
    ro, _ = orc.batched_forward(qq, kk, vv, lams)
    (rdq, rdk, rdv), _ = orc.batched_backward(qq, kk, vv, do, lams)
    for name, got, ref in (("o", o, ro), ("dq", tq.grad, rdq), ("dk", tk.grad, rdk), ("dv", tv.grad, rdv)):
        _check(got, ref, torch.float32, name)
    # the default route is the split pass: bit-identical to forcing it (the kernels are deterministic)
    assert torch.equal(o.detach(), ops.la_forward(tq.detach(), tk.detach(), tv.detach(), lams, backend="tcgen05"))


@pytest.mark.parametrize("dtype", DTYPES, ids=IDS)
@pytest.mark.parametrize("d", [64, 128])
def test_state_passes_and_resume(dtype, d):
    """la_fwd_state + la_fwd_ex(RESUME) == la_fwd and la_bwd_state + la_bwd_ex(RESUME, dkdv) == la_bwd's
    dK / dV sweep, bitwise, on the tensor-core passes (bf16, and the fp32 split pass whose summaries are
    whole segments); the summary itself is the oracle's F(n) with kv_in = 0."""
    b, h, n = 1, 3, 3000
    lams = [0.9999, 0.99, 0.4]
    q, k, v, do = (_dev(a, dtype) for a in _inputs((b, h, n, d), 71 + d))
    kv_in = torch.rand(b, h, d, d, device=DEV) * 0.01
    ws = ops.new_workspace((b, h, n, d), dtype)
    delta = ops.la_forward_state(k, v, lams, workspace=ws)
    (o_r, kv_r), seg_r = ops.la_forward(q, k, v, lams, kv_in=kv_in, want_state=True, want_seg_states=True,
                                        workspace=ws, resume=True)
    (o, kv), seg = ops.la_forward(q, k, v, lams, kv_in=kv_in, want_state=True, want_seg_states=True)
    assert torch.equal(o_r, o) and torch.equal(kv_r, kv)
    assert (seg is None and seg_r is None) or torch.equal(seg_r, seg)
    _, rkv0 = orc.batched_forward(_host(q), _host(k), _host(v), lams)
    _check(delta, rkv0, dtype, "forward summary")
    ws2 = ops.new_workspace((b, h, n, d), dtype)
    ops.la_backward_state(q, do, lams, workspace=ws2)
    dkv_in = torch.rand(b, h, d, d, device=DEV) * 0.01
    _, dk_r, dv_r, dkv_r = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, dkv_in=dkv_in, parts="dkdv",
                                           want_state=True, workspace=ws2, resume=True)
    dq, dk, dv, dkv = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, dkv_in=dkv_in, want_state=True,
                                      fwd_seg_states=seg)
    assert torch.equal(dk_r, dk) and torch.equal(dv_r, dv) and torch.equal(dkv_r, dkv)
    (rdq, rdk, rdv), rdkv = orc.batched_backward(_host(q), _host(k), _host(v), _host(do), lams, kv_in=_host(kv_in),
                                                 dkv_in=_host(dkv_in))
    for name, got, ref in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv), ("dkv", dkv, rdkv)):
        _check(got, ref, dtype, f"{name} d={d}")
