"""Parity of the fp32 tensor-core pass (la_tc32.cu: three-term bf16 split on tcgen05) with the oracle.

Tolerance: the north star's fp32 bar, <= 1e-4 per-entry relative on positive uniform(0.05, 1)
inputs (``max_rel_error``), and <= 1e-5 ``max_scaled_error`` on standard-normal inputs -- the same
bars the SIMT fp32 path meets (test_gpu_parity.py).  The oracle (fp64 restatement of kernels.py:253-334,
pinned to the reference by tests/test_oracle.py) runs on the exact fp32 operands the device saw.
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
TOL = 1e-4


def _inputs(shape, seed, dist="pos", count=4):
    rng = np.random.default_rng(seed)
    if dist == "pos":
        return [rng.uniform(0.05, 1.0, shape) for _ in range(count)]
    return [rng.standard_normal(shape) for _ in range(count)]


def _dev(a):
    return torch.tensor(a, dtype=torch.float32, device=DEV)


def _host(t):
    return t.detach().double().cpu().numpy()


def _check(got, ref, dist, what):
    metric = orc.max_rel_error if dist == "pos" else orc.max_scaled_error
    tol = TOL if dist == "pos" else 1e-5
    err = metric(_host(got), ref)
    assert err <= tol, f"{what}: {err:.3e} > {tol:g}"
    return err


def _run(b, h, n, lams, seed, dist="pos", segments=0, backend="tcgen05", layout="bhnd"):
    q, k, v, do = _inputs((b, h, n, 128), seed, dist)
    tq, tk, tv, tdo = (_dev(a) for a in (q, k, v, do))
    if layout == "bnhd":
        tq, tk, tv, tdo = (t.transpose(1, 2).contiguous().transpose(1, 2) for t in (tq, tk, tv, tdo))
    o = ops.la_forward(tq, tk, tv, lams, backend=backend, segments=segments)
    dq, dk, dv = ops.la_backward(tq, tk, tv, tdo, lams, backend=backend, segments=segments)
    qq, kk, vv, dd = (_host(t) for t in (tq, tk, tv, tdo))
    ro, _ = orc.batched_forward(qq, kk, vv, lams)
    (rdq, rdk, rdv), _ = orc.batched_backward(qq, kk, vv, dd, lams)
    for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        _check(got, ref, dist, f"{name} n={n} seg={segments} {dist}")


LAMS3 = [1.0, 0.999, 0.9]
LAMS_STRONG = [0.5, 0.05, 5.5e-4]


@pytest.mark.parametrize("n", [1, 2, 5, 127, 128, 129, 255, 300, 1000])
def test_tc32_ragged_lengths(n):
    _run(2, 3, n, LAMS3, seed=n)


@pytest.mark.parametrize("segments", [1, 2, 3, 7])
def test_tc32_forced_segments(segments):
    _run(1, 3, 1500, LAMS3, seed=11, segments=segments)
    _run(1, 3, 1500, LAMS_STRONG, seed=12, segments=segments)


def test_tc32_strong_decays_and_normal_inputs():
    _run(2, 3, 700, LAMS_STRONG, seed=3)
    _run(2, 3, 700, LAMS3, seed=4, dist="normal")


def test_tc32_model_native_layout():
    _run(2, 3, 400, LAMS3, seed=5, layout="bnhd")


def test_tc32_matches_simt_backend():
    """The two fp32 backends agree to the fp32 bar (both are <= 1e-4 from the oracle)."""
    q, k, v, do = (_dev(a) for a in _inputs((1, 4, 777, 128), 21))
    lams = [1.0, 0.99, 0.9, 0.3]
    o_tc = ops.la_forward(q, k, v, lams, backend="tcgen05")
    o_si = ops.la_forward(q, k, v, lams, backend="simt")
    g_tc = ops.la_backward(q, k, v, do, lams, backend="tcgen05")
    g_si = ops.la_backward(q, k, v, do, lams, backend="simt")
    assert orc.max_rel_error(_host(o_tc), _host(o_si)) <= 2 * TOL
    for a, b_ in zip(g_tc, g_si):
        assert orc.max_rel_error(_host(a), _host(b_)) <= 2 * TOL


def test_tc32_state_chaining():
    """kv_in / kv_out and dkv_in / dkv_out: two halves chained equal the whole (and the oracle's states)."""
    b, h, n = 1, 2, 900
    lams = [0.999, 0.95]
    q, k, v, do = _inputs((b, h, n, 128), 31)
    kv0, dkv0 = (np.random.default_rng(32).uniform(0.0, 0.5, (b, h, 128, 128)) for _ in range(2))
    tq, tk, tv, tdo = (_dev(a) for a in (q, k, v, do))
    o, kv = ops.la_forward(tq, tk, tv, lams, kv_in=_dev(kv0), want_state=True, backend="tcgen05")
    dq, dk, dv, dkv = ops.la_backward(tq, tk, tv, tdo, lams, kv_in=_dev(kv0), dkv_in=_dev(dkv0), want_state=True,
                                      backend="tcgen05")
    qq, kk, vv, dd = (_host(t) for t in (tq, tk, tv, tdo))
    kv0f, dkv0f = _host(_dev(kv0)), _host(_dev(dkv0))
    ro, rkv = orc.batched_forward(qq, kk, vv, lams, kv_in=kv0f)
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, lams, kv_in=kv0f, dkv_in=dkv0f)
    for name, got, ref in (("o", o, ro), ("kv", kv, rkv), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv),
                           ("dkv", dkv, rdkv)):
        _check(got, ref, "pos", name)


def test_tc32_autograd_default_backend():
    """fp32 at d = 128 routes to the tensor cores by default; the autograd op saves segment states."""
    b, h, n = 1, 4, 2000  # bh = 4: the plan splits each sequence into segments
    lams = [1.0, 0.99, 0.9, 0.5]
    q, k, v, do = _inputs((b, h, n, 128), 41)
    tq, tk, tv = (_dev(a).requires_grad_(True) for a in (q, k, v))
    o = lightning_attention(tq, tk, tv, lams)
    o.backward(_dev(do))
    ro, _ = orc.batched_forward(*(_host(t) for t in (tq, tk, tv)), lams)
    (rdq, rdk, rdv), _ = orc.batched_backward(*(_host(t) for t in (tq, tk, tv)), _host(_dev(do)), lams)
    for name, got, ref in (("o", o, ro), ("dq", tq.grad, rdq), ("dk", tk.grad, rdk), ("dv", tv.grad, rdv)):
        _check(got, ref, "pos", name)


def test_tc32_tnl1b_heads_long():
    """TNL-1B heads (H = 16, decay_rate(h, 1, 16, 16) down to 5.5e-4) at n = 16384, sampled heads."""
    b, h, n = 1, 16, 16384
    lams = [orc.decay_rate(j + 1, 1, 16, 16) for j in range(h)]
    rng = np.random.default_rng(51)
    tq, tk, tv, tdo = (torch.rand((b, h, n, 128), generator=torch.Generator().manual_seed(51 + s),
                                  dtype=torch.float32).mul_(0.95).add_(0.05).to(DEV) for s in range(4))
    o = ops.la_forward(tq, tk, tv, lams)
    dq, dk, dv = ops.la_backward(tq, tk, tv, tdo, lams)
    for j in sorted({0, int(rng.integers(1, 15)), 15}):
        qq, kk, vv, dd = (_host(t[0, j]) for t in (tq, tk, tv, tdo))
        ro = orc.tiled_forward(qq, kk, vv, lams[j])
        rdq, rdk, rdv = orc.tiled_backward(qq, kk, vv, dd, lams[j])
        for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
            _check(got[0, j], ref, "pos", f"{name} head {j}")
