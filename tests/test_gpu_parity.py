"""Parity of the CUDA path with the oracle / the reference's golden outputs.

Tolerances (north star, stated per test): fp64 <= 1e-10 relative, fp32 <=
1e-4 relative, bf16 operands with fp32 accumulation <= 2e-2 relative -- all
per-entry ``max_rel_error`` on positive uniform(0.05, 1) inputs, and
``max_scaled_error`` on standard-normal inputs (oracles.py:53-81).
"""

import numpy as np
import pytest

from conftest import case_inputs, config1_inputs, golden_array, golden_cases, golden_config1
from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2405_17381_b200 import lightning_attention, ops  # noqa: E402

DEV = torch.device("cuda", 0)
TOL = {torch.float64: 1e-10, torch.float32: 1e-4, torch.bfloat16: 2e-2}
CASES = golden_cases()


def dev(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).to(DEV).to(dtype)


def host(t):
    return t.detach().to(torch.float64).cpu().numpy()


def rounded(a, dtype):
    """The operand values the device actually sees (bf16/fp32 rounding of the fp64 input)."""
    return host(dev(a, dtype))


# --------------------------------------------------------------------------
# golden vectors produced by the real reference
# --------------------------------------------------------------------------


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_golden_cases(case, dtype):
    name, n, d, B, lam, seed, dist = case
    q, k, v, do = case_inputs(n, d, seed, dist)
    tq, tk, tv, tdo = (dev(a, dtype)[None, None] for a in (q, k, v, do))
    o = ops.la_forward(tq, tk, tv, lam, block=B)
    dq, dk, dv = ops.la_backward(tq, tk, tv, tdo, lam, block=B)
    metric = orc.max_rel_error if dist == "pos" else orc.max_scaled_error
    tol = TOL[dtype] if dist == "pos" else (1e-13 if dtype == torch.float64 else 1e-5)
    for key, got in (("o64", o), ("dq64", dq), ("dk64", dk), ("dv64", dv)):
        g = host(got)[0, 0]
        ref, view = golden_array(f"{name}/{key}", g)
        err = metric(view(g), ref)
        assert err <= tol, f"{name} {key} {dtype}: {err:.3e} > {tol:g}"


def test_config1_fp32_and_fp64():
    """BASELINE.json configs[0]: batch=1, H=4, n=1024, d=64, B=64, fp32, per-head decay."""
    c = golden_config1()
    q, k, v, do = config1_inputs()
    for dtype in (torch.float32, torch.float64):
        tq, tk, tv, tdo = (dev(a, dtype) for a in (q, k, v, do))
        o = host(lightning_attention(tq, tk, tv, c["lams"], c["B"]))
        dq, dk, dv = (host(t) for t in ops.la_backward(tq, tk, tv, tdo, c["lams"], block=c["B"]))
        for h in range(c["H"]):
            for key, arr in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
                ref, view = golden_array(f"config1/h{h}/{key}64", arr[0, h])
                err = orc.max_rel_error(view(arr[0, h]), ref)
                assert err <= TOL[dtype], f"h={h} {key} {dtype}: {err:.3e}"
        # the stored goldens are compressed (row sums + every 97th entry): also compare every entry against
        # the oracle (pinned to the reference by tests/test_oracle.py) on the same inputs
        ro, _ = orc.batched_forward(q, k, v, c["lams"], c["B"])
        (rdq, rdk, rdv), _ = orc.batched_backward(q, k, v, do, c["lams"], c["B"])
        for key, arr, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
            err = orc.max_rel_error(arr, ref)
            assert err <= TOL[dtype], f"full {key} {dtype}: {err:.3e}"


# --------------------------------------------------------------------------
# batched op: layouts, per-head decay, segments, carried states
# --------------------------------------------------------------------------


def _batched(b, h, n, d, seed, dist="pos"):
    rng = np.random.default_rng(seed)
    if dist == "pos":
        return [rng.uniform(0.05, 1.0, (b, h, n, d)) for _ in range(4)]
    return [rng.standard_normal((b, h, n, d)) / np.sqrt(d) for _ in range(4)]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16], ids=["f64", "f32", "bf16"])
@pytest.mark.parametrize("shape", [(2, 3, 77, 16), (1, 2, 300, 64), (2, 2, 257, 128), (1, 1, 1, 8)])
@pytest.mark.parametrize("backend", ["simt", "auto"])
def test_batched_forward_backward(shape, dtype, backend):
    b, h, n, d = shape
    lams = [1.0, 0.9, 0.5][:h]
    q, k, v, do = _batched(b, h, n, d, seed=n + d)
    qq, kk, vv, dd = (rounded(a, dtype) for a in (q, k, v, do))
    ro, rkv = orc.batched_forward(qq, kk, vv, lams)
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, lams)
    tq, tk, tv, tdo = (dev(a, dtype) for a in (q, k, v, do))
    o, kv = ops.la_forward(tq, tk, tv, lams, want_state=True, backend=backend)
    dq, dk, dv, dkv = ops.la_backward(tq, tk, tv, tdo, lams, want_state=True, backend=backend)
    tol = TOL[dtype]
    for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv),
                           ("kv_out", kv, rkv), ("dkv_out", dkv, rdkv)):
        err = orc.max_rel_error(host(got), ref)
        assert err <= tol, f"{name}: {err:.3e} > {tol:g}"


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_sign_mixed_scaled_error(dtype):
    b, h, n, d = 2, 2, 640, 128
    lams = [0.99, 0.8]
    q, k, v, do = _batched(b, h, n, d, seed=3, dist="normal")
    qq, kk, vv, dd = (rounded(a, dtype) for a in (q, k, v, do))
    ro, _ = orc.batched_forward(qq, kk, vv, lams)
    (rdq, rdk, rdv), _ = orc.batched_backward(qq, kk, vv, dd, lams)
    tq, tk, tv, tdo = (dev(a, dtype) for a in (q, k, v, do))
    o = ops.la_forward(tq, tk, tv, lams)
    grads = ops.la_backward(tq, tk, tv, tdo, lams)
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    for got, ref in zip((o,) + tuple(grads), (ro, rdq, rdk, rdv)):
        assert orc.max_scaled_error(host(got), ref) <= tol


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_layout_bnhd_equals_bhnd(dtype):
    b, h, n, d = 2, 4, 200, 128
    lams = [1.0, 0.99, 0.9, 0.5]
    q, k, v, do = (dev(a, dtype) for a in _batched(b, h, n, d, seed=7))
    o = ops.la_forward(q, k, v, lams)
    grads = ops.la_backward(q, k, v, do, lams)
    t = lambda x: x.transpose(1, 2).contiguous()  # noqa: E731
    o2 = ops.la_forward(t(q), t(k), t(v), lams, layout="bnhd")
    grads2 = ops.la_backward(t(q), t(k), t(v), t(do), lams, layout="bnhd")
    assert torch.equal(o, o2.transpose(1, 2))
    for a, b2 in zip(grads, grads2):
        assert torch.equal(a, b2.transpose(1, 2))


@pytest.mark.parametrize("backend", ["simt", "auto"])
@pytest.mark.parametrize("segments", [1, 2, 3, 7])
def test_segment_split_is_exact(segments, backend):
    """The intra-GPU sequence split (state summaries + decayed scan) changes nothing but rounding."""
    dtype = torch.bfloat16 if backend == "auto" else torch.float32
    b, h, n, d = 1, 2, 1000, 128
    lams = [0.999, 0.95]
    q, k, v, do = _batched(b, h, n, d, seed=11)
    qq, kk, vv, dd = (rounded(a, dtype) for a in (q, k, v, do))
    ro, _ = orc.batched_forward(qq, kk, vv, lams)
    (rdq, rdk, rdv), _ = orc.batched_backward(qq, kk, vv, dd, lams)
    tq, tk, tv, tdo = (dev(a, dtype) for a in (q, k, v, do))
    o, seg = ops.la_forward(tq, tk, tv, lams, segments=segments, backend=backend, want_seg_states=True)
    assert (seg is None) == (segments == 1)
    grads = ops.la_backward(tq, tk, tv, tdo, lams, segments=segments, backend=backend)
    grads_saved = ops.la_backward(tq, tk, tv, tdo, lams, segments=segments, backend=backend, fwd_seg_states=seg)
    for got, ref in zip((o,) + tuple(grads), (ro, rdq, rdk, rdv)):
        assert orc.max_rel_error(host(got), ref) <= TOL[dtype]
    # the forward's segment states reproduce the recomputed ones up to fp32 summation order
    # (an output can land one bf16 ulp = 2^-7 relative apart); both meet the bar vs the oracle
    for a, b, ref in zip(grads, grads_saved, (rdq, rdk, rdv)):
        assert orc.max_rel_error(host(a), host(b)) <= (1e-5 if dtype == torch.float32 else 1e-2)
        assert orc.max_rel_error(host(b), ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16], ids=["f64", "f32", "bf16"])
def test_state_chaining_matches_whole_sequence(dtype):
    """kv_out -> kv_in and dkv_out -> dkv_in chain two halves into the whole (the SP contract)."""
    b, h, n, d = 1, 3, 700, 128 if dtype != torch.float64 else 32
    lams = [1.0, 0.97, 0.6]
    q, k, v, do = (dev(a, dtype) for a in _batched(b, h, n, d, seed=5))
    cut = 384
    whole = ops.la_forward(q, k, v, lams)
    wgrads = ops.la_backward(q, k, v, do, lams)
    sl = lambda x, a, z: x[:, :, a:z].contiguous()  # noqa: E731
    o1, kv1 = ops.la_forward(sl(q, 0, cut), sl(k, 0, cut), sl(v, 0, cut), lams, want_state=True)
    o2 = ops.la_forward(sl(q, cut, n), sl(k, cut, n), sl(v, cut, n), lams, kv_in=kv1)
    g2 = ops.la_backward(sl(q, cut, n), sl(k, cut, n), sl(v, cut, n), sl(do, cut, n), lams, kv_in=kv1,
                         want_state=True)
    g1 = ops.la_backward(sl(q, 0, cut), sl(k, 0, cut), sl(v, 0, cut), sl(do, 0, cut), lams, dkv_in=g2[3])
    tol = TOL[dtype]
    assert orc.max_rel_error(host(torch.cat([o1, o2], 2)), host(whole)) <= tol
    for a, b2, w in zip(g1, g2[:3], wgrads):
        assert orc.max_rel_error(host(torch.cat([a, b2], 2)), host(w)) <= tol
    # the exported local summaries compose the same way
    d1 = ops.la_forward_state(sl(k, 0, cut), sl(v, 0, cut), lams)
    assert orc.max_rel_error(host(d1), host(kv1)) <= tol
    dd2 = ops.la_backward_state(sl(q, cut, n), sl(do, cut, n), lams)
    assert orc.max_rel_error(host(dd2), host(g2[3])) <= tol


@pytest.mark.parametrize("segments", [0, 1, 3])
def test_backward_with_edge_states_and_saved_segment_states(segments):
    """The backward's concurrent schedule (dq pass beside the dK/dV chain) with kv_in, dkv_in, dkv_out and
    the forward's segment states: the same gradients and dkv_out as the sequential recomputation."""
    b, h, n, d = 2, 3, 1500, 128
    lams = [1.0, 0.97, 0.6]
    q, k, v, do = (dev(a, torch.bfloat16) for a in _batched(b, h, n, d, seed=9))
    kv_in = torch.randn(b, h, d, d, device="cuda") * 0.05
    dkv_in = torch.randn(b, h, d, d, device="cuda") * 0.05
    o, seg = ops.la_forward(q, k, v, lams, kv_in=kv_in, segments=segments, want_seg_states=True)
    want = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, dkv_in=dkv_in, segments=segments, want_state=True)
    got = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, dkv_in=dkv_in, segments=segments, want_state=True,
                          fwd_seg_states=seg)
    for a, w in zip(got[:3], want[:3]):
        assert orc.max_rel_error(host(a), host(w)) <= 1e-2
    assert orc.max_rel_error(host(got[3]), host(want[3])) <= 1e-5
    # and against the oracle run on the same bf16 inputs with the same edge states
    qq, kk, vv, dd = (host(t) for t in (q, k, v, do))
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, lams, kv_in=host(kv_in), dkv_in=host(dkv_in))
    for a, r in zip(got[:3], (rdq, rdk, rdv)):
        assert orc.max_rel_error(host(a), r) <= TOL[torch.bfloat16]


def test_multi_wave_units_with_edge_states():
    """More (batch, head) units than one wave (185 CTAs on 148 SMs, two waves of one-unit CTAs) and an
    unsplit, ragged sequence: every CTA loads its own unit's kv_in / dkv_in and exports its kv_out /
    dkv_out."""
    b, h, n, d = 37, 5, 300, 128  # bh = 185 > 148: 95 CTAs, 1-2 units each
    lams = [1.0, 0.99, 0.9, 0.7, 0.5]
    q, k, v, do = (dev(a, torch.bfloat16) for a in _batched(b, h, n, d, seed=21))
    kv_in = torch.randn(b, h, d, d, device="cuda") * 0.05
    dkv_in = torch.randn(b, h, d, d, device="cuda") * 0.05
    assert ops.segment_count(ops._desc(ops._geometry(q, "bhnd"), q.dtype, None, "auto", 0)) == 1
    o, kv_out = ops.la_forward(q, k, v, lams, kv_in=kv_in, want_state=True)
    dq, dk, dv, dkv_out = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, dkv_in=dkv_in, want_state=True)
    qq, kk, vv, dd = (host(t) for t in (q, k, v, do))
    ro, rkv = orc.batched_forward(qq, kk, vv, lams, kv_in=host(kv_in))
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, lams, kv_in=host(kv_in), dkv_in=host(dkv_in))
    tol = TOL[torch.bfloat16]
    for got, ref in ((o, ro), (kv_out, rkv), (dq, rdq), (dk, rdk), (dv, rdv), (dkv_out, rdkv)):
        assert orc.max_rel_error(host(got), ref) <= tol


@pytest.mark.parametrize("n", [1, 2, 127, 129, 255])
def test_tcgen05_tiny_and_ragged_lengths(n):
    """The tensor-core path at lengths shorter than / just around one 128-row chunk (TMA boxes past the
    end read zeros and store nothing), with kv_in and every edge state exported."""
    b, h, d = 2, 3, 128
    lams = [1.0, 0.9, 0.5]
    q, k, v, do = (dev(a, torch.bfloat16) for a in _batched(b, h, n, d, seed=100 + n))
    kv_in = torch.rand(b, h, d, d, device="cuda") * 0.05
    o, kv_out = ops.la_forward(q, k, v, lams, kv_in=kv_in, want_state=True, backend="tcgen05")
    dq, dk, dv, dkv_out = ops.la_backward(q, k, v, do, lams, kv_in=kv_in, want_state=True, backend="tcgen05")
    qq, kk, vv, dd = (host(t) for t in (q, k, v, do))
    ro, rkv = orc.batched_forward(qq, kk, vv, lams, kv_in=host(kv_in))
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, lams, kv_in=host(kv_in))
    for got, ref in ((o, ro), (kv_out, rkv), (dq, rdq), (dk, rdk), (dv, rdv), (dkv_out, rdkv)):
        assert orc.max_rel_error(host(got), ref) <= TOL[torch.bfloat16]


def test_autograd_function_matches_ops():
    b, h, n, d = 2, 2, 333, 128
    lams = [0.9, 0.99]
    q, k, v, do = (dev(a, torch.bfloat16) for a in _batched(b, h, n, d, seed=9))
    leaves = [t.clone().requires_grad_(True) for t in (q, k, v)]
    o = lightning_attention(*leaves, lams)
    o.backward(do)
    assert torch.equal(o.detach(), ops.la_forward(q, k, v, lams))
    for leaf, g in zip(leaves, ops.la_backward(q, k, v, do, lams)):
        assert torch.equal(leaf.grad, g)


def test_errors_raise_reference_exceptions():
    from paper_2405_17381_b200.errors import DomainError, ShapeError

    q = torch.zeros(1, 2, 8, 16, device=DEV)
    with pytest.raises(ShapeError):
        ops.la_forward(q, q, q[:, :1], [0.5, 0.5])
    with pytest.raises(DomainError):
        ops.la_forward(q, q, q, [0.5, 1.5])
    with pytest.raises(ShapeError):
        ops.la_forward(q, q, q, [0.5, 0.5, 0.5])
    with pytest.raises(DomainError):
        ops.la_forward(q, q, q, 0.5, block=0)
    with pytest.raises(DomainError):
        ops.la_forward(q.cpu(), q.cpu(), q.cpu(), 0.5)


# --------------------------------------------------------------------------
# full-size properties (BASELINE sizes; the oracle cannot finish these)
# --------------------------------------------------------------------------


@pytest.mark.parametrize("n", [8192, 131072])
def test_full_size_properties(n):
    """TNL-1B head shape at long n: segment split == unsplit, linearity in v, two-halves chaining."""
    b, h, d = 1, 2, 128
    lams = [0.9996, 0.97]
    g = torch.Generator(device=DEV).manual_seed(n)
    q, k, v, v2 = (torch.randn(b, h, n, d, device=DEV, generator=g, dtype=torch.float32) / d ** 0.5
                   for _ in range(4))
    qb, kb, vb, v2b = (t.to(torch.bfloat16) for t in (q, k, v, v2))
    o_auto = ops.la_forward(qb, kb, vb, lams).float()
    o_one = ops.la_forward(qb, kb, vb, lams, segments=1).float()
    scale = o_one.abs().max()
    assert ((o_auto - o_one).abs().max() / scale).item() <= 2e-2
    # linearity in v (fp32 path, exact up to rounding)
    oa = ops.la_forward(q, k, v, lams)
    ob = ops.la_forward(q, k, v2, lams)
    oab = ops.la_forward(q, k, 2.0 * v + v2, lams)
    assert ((oab - (2.0 * oa + ob)).abs().max() / oab.abs().max()).item() <= 1e-5
    # chaining halves through kv_in reproduces the whole (bf16 path)
    cut = n // 2
    sl = lambda x, a, z: x[:, :, a:z].contiguous()  # noqa: E731
    _, kv1 = ops.la_forward(sl(qb, 0, cut), sl(kb, 0, cut), sl(vb, 0, cut), lams, want_state=True)
    o2 = ops.la_forward(sl(qb, cut, n), sl(kb, cut, n), sl(vb, cut, n), lams, kv_in=kv1).float()
    assert ((o2 - o_auto[:, :, cut:]).abs().max() / scale).item() <= 2e-2


def test_saved_segment_states_are_validated():
    """fwd_seg_states from another problem (other plan, dtype or layout) is refused, not misread."""
    from paper_2405_17381_b200.errors import ShapeError
    b, h, n, d = 1, 2, 4096, 128
    q, k, v, do = (torch.rand(b, h, n, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    _, seg = ops.la_forward(q, k, v, [0.9, 0.99], want_seg_states=True)
    assert seg is not None
    with pytest.raises(ShapeError):
        ops.la_backward(q, k, v, do, [0.9, 0.99], fwd_seg_states=seg[:, :, :-1])
    with pytest.raises(ShapeError):
        ops.la_backward(q, k, v, do, [0.9, 0.99], fwd_seg_states=seg.double())
    with pytest.raises(ShapeError):
        ops.la_backward(q, k, v, do, [0.9, 0.99], fwd_seg_states=seg.transpose(3, 4))


@pytest.mark.parametrize("n", [5000, 12345, 33333])
def test_long_ragged_segmented_sequences(n):
    """Long sequences whose length is no multiple of the chunk, segment or sub-segment length (the
    planner splits them; every boundary is ragged), forward + backward with saved segment states."""
    b, h, d = 1, 2, 128
    lams = [0.999, 0.9]
    q, k, v, do = (dev(a, torch.bfloat16) for a in _batched(b, h, n, d, seed=n))
    assert ops.segment_count(ops._desc(ops._geometry(q, "bhnd"), q.dtype, None, "auto", 0)) > 1
    (o, kv_out), seg = ops.la_forward(q, k, v, lams, want_state=True, want_seg_states=True)
    dq, dk, dv, dkv_out = ops.la_backward(q, k, v, do, lams, want_state=True, fwd_seg_states=seg)
    qq, kk, vv, dd = (host(t) for t in (q, k, v, do))
    ro, rkv = orc.batched_forward(qq, kk, vv, lams)
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, lams)
    for got, ref in ((o, ro), (kv_out, rkv), (dq, rdq), (dk, rdk), (dv, rdv), (dkv_out, rdkv)):
        assert orc.max_rel_error(host(got), ref) <= TOL[torch.bfloat16]


def test_grid_limit_batch_heads():
    """batch * heads at the grid limit (65535 (batch, head) rows of CTAs): sampled sequences match the
    oracle; one more is refused with the unsupported status, not launched."""
    b, h, n, d = 16383, 4, 3, 128
    rng = np.random.default_rng(77)
    q, k, v, do = (torch.as_tensor(rng.uniform(0.05, 1.0, (b, h, n, d)), dtype=torch.bfloat16, device="cuda")
                   for _ in range(4))
    lams = [0.9, 0.5, 1.0, 0.99]
    o = ops.la_forward(q, k, v, lams)
    dq, dk, dv = ops.la_backward(q, k, v, do, lams)
    for bi in (0, 4097, b - 1):
        sl = lambda t: host(t[bi:bi + 1])  # noqa: E731
        ro, _ = orc.batched_forward(sl(q), sl(k), sl(v), lams)
        (rdq, rdk, rdv), _ = orc.batched_backward(sl(q), sl(k), sl(v), sl(do), lams)
        for got, ref in ((o, ro), (dq, rdq), (dk, rdk), (dv, rdv)):
            assert orc.max_rel_error(sl(got), ref) <= TOL[torch.bfloat16]
    from paper_2405_17381_b200._lib import UnsupportedError
    q2 = torch.zeros(16384, 4, n, d, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(UnsupportedError):
        ops.la_forward(q2, q2, q2, lams)


def test_misaligned_states_rejected_by_the_abi_and_realigned_by_ops():
    """The C ABI refuses state buffers that are not 16-byte aligned (the kernels read them as 16-byte
    vectors); the Python layer copies such a state instead of passing it through."""
    import ctypes
    from paper_2405_17381_b200 import _lib
    b, h, n, d = 1, 2, 256, 128
    q, k, v = (torch.rand(b, h, n, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    buf = torch.zeros(b * h * d * d + 1, device="cuda")
    kv_off = buf[1:].view(b, h, d, d)  # 4 bytes past an aligned base
    assert kv_off.data_ptr() % 16 == 4
    lib = _lib.load()
    desc = ops._desc(ops._geometry(q, "bhnd"), q.dtype, None, "auto", 0)
    lam = ops.decay_tensor([0.9, 0.5], h, q.device)
    o = torch.empty_like(q)
    ws, nbytes = ops._workspace(lib, desc, q.device)
    rc = lib.la_fwd(ctypes.byref(desc), ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
                    ctypes.c_void_p(v.data_ptr()), ctypes.cast(ctypes.c_void_p(lam.data_ptr()),
                                                                ctypes.POINTER(ctypes.c_double)),
                    ctypes.c_void_p(kv_off.data_ptr()), ctypes.c_void_p(o.data_ptr()), None, None,
                    ctypes.c_void_p(ws.data_ptr()), nbytes, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == _lib.LA_ERR_SHAPE and b"aligned" in lib.la_last_error()
    kv_ok = kv_off.clone()
    kv_off.copy_(torch.rand_like(kv_off) * 0.05)
    kv_ok.copy_(kv_off)
    assert torch.equal(ops.la_forward(q, k, v, [0.9, 0.5], kv_in=kv_off), ops.la_forward(q, k, v, [0.9, 0.5], kv_in=kv_ok))
