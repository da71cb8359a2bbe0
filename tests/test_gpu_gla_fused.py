"""The fused GLA core forward (la_gla_core_fwd, §8(f) rank 1): act + LRPE applied to each q / k tile in
the tcgen05 pass kernel's shared memory.

Checked against a torch fp64 restatement of model.py:381-397 (act, model.py:60-99; LRPE,
positional.py:126-150) and the decayed causal left product (oracles.py:100) on the same bf16 inputs:
  * q_out / k_out (the transformed rows) within 1.5e-2 scaled -- one bf16 rounding of the result on top of
    the hardware tanh / sincos approximations;
  * o within 2e-2 scaled (the north star's bf16 bar), and within 2e-2 of the two-step path
    (la_gla_prologue + la_fwd) it replaces;
  * the whole bf16 GLA layer through autograd on the fused path within tests/test_gpu_gla.py's bf16 bars.
"""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle.linattn_oracle import decay_rate  # noqa: E402
from paper_2405_17381_b200 import ops  # noqa: E402
from paper_2405_17381_b200._lib import UnsupportedError  # noqa: E402

DEV = torch.device("cuda", 0)
H, D = 16, 128
THETA = torch.tensor([10000.0 ** (-2.0 * j / D) for j in range(D // 2)], dtype=torch.float64, device=DEV)


def _act64(z, act):
    if act == "swish":
        return z * torch.sigmoid(z)
    if act == "one_plus_elu":
        return torch.where(z > 0, z + 1, torch.exp(torch.clamp(z, max=0)))
    return z


def _rot64(z, theta, offset):
    b, n, w = z.shape
    pos = torch.arange(offset, offset + n, dtype=torch.float64, device=z.device)
    ang = pos[:, None] * theta[None, :]
    c, s = torch.cos(ang)[None, :, None, :], torch.sin(ang)[None, :, None, :]
    z = z.view(b, n, w // D, D // 2, 2)
    z1, z2 = z[..., 0], z[..., 1]
    return torch.stack((z1 * c - z2 * s, z1 * s + z2 * c), -1).view(b, n, w)


def _attn64(q, k, v, lams, kv_in=None):
    """Decayed causal attention as the left product (+ the entering state's term), [b, n, H*D] rows."""
    b, n, w = q.shape
    qh, kh, vh = (t.double().view(b, n, H, D).transpose(1, 2) for t in (q, k, v))
    lam = torch.tensor(lams, dtype=torch.float64, device=q.device)
    t = torch.arange(n, device=q.device)
    diff = (t[:, None] - t[None, :]).to(torch.float64)
    mask = torch.where(diff[None] >= 0, lam[:, None, None] ** diff.clamp(min=0)[None], torch.zeros((), device=q.device,
                                                                                                   dtype=torch.float64))
    a = ((qh @ kh.transpose(-1, -2)) * mask[None]) @ vh
    if kv_in is not None:
        a = a + (lam[None, :, None, None] ** (t.double() + 1)[None, None, :, None]) * (qh @ kv_in.double())
    return a.transpose(1, 2).reshape(b, n, w)


def _scaled(got, want):
    return ((got.double() - want).abs().max() / want.abs().max().clamp(min=1e-30)).item()


def _inputs(b, n, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return [(torch.randn(b, n, H * D, device=DEV, generator=g) * sc).to(torch.bfloat16) for sc in (1.0, 1.0, 0.5)]


LAMS = [decay_rate(h, 1, H, 16) for h in range(1, H)] + [1.0]


@pytest.mark.parametrize("act,rot,offset", [("swish", True, 0), ("swish", False, 0), ("one_plus_elu", True, 37),
                                            ("none", True, 5), ("one_plus_elu", False, 0)])
def test_fused_core_matches_fp64(act, rot, offset):
    b, n = 6, 777  # batch * heads = 96: one unsegmented wave; n ragged (tail chunk of 9 rows)
    qp, kp, v = _inputs(b, n, 7)
    theta = THETA if rot else None
    o, q, k = ops.gla_core_forward(qp, kp, v, LAMS, H, act=act, theta=theta, offset=offset)
    q64, k64 = (_act64(t.double(), act) for t in (qp, kp))
    if rot:
        q64, k64 = _rot64(q64, THETA, offset), _rot64(k64, THETA, offset)
    assert _scaled(q, q64) <= 1.5e-2
    assert _scaled(k, k64) <= 1.5e-2
    assert _scaled(o, _attn64(q64, k64, v, LAMS)) <= 2e-2
    # the attention itself on the kernel's own transformed operands (tighter: no prologue rounding inside)
    assert _scaled(o, _attn64(q, k, v, LAMS)) <= 1e-2
    # the two-step path it replaces
    q2, k2 = ops.gla_prologue(qp, kp, H, act=act, theta=theta, offset=offset)
    o2 = ops.la_forward(*(t.view(b, n, H, D) for t in (q2, k2, v)), LAMS, layout="bnhd").view(b, n, H * D)
    assert _scaled(o, o2.double()) <= 2e-2


def test_fused_core_states_and_no_qk():
    """kv_in / kv_out as la_fwd; want_qk=False (inference) gives the same o."""
    b, n = 6, 512
    qp, kp, v = _inputs(b, n, 11)
    kv_in = torch.rand(b, H, D, D, device=DEV) * 0.1
    o, q, k, kv = ops.gla_core_forward(qp, kp, v, LAMS, H, theta=THETA, kv_in=kv_in, want_state=True)
    o_nq, qn, kn = ops.gla_core_forward(qp, kp, v, LAMS, H, theta=THETA, kv_in=kv_in, want_qk=False)
    assert qn is None and kn is None
    assert torch.equal(o, o_nq)
    o2, kv2 = ops.la_forward(*(t.view(b, n, H, D) for t in (q, k, v)), LAMS, layout="bnhd", kv_in=kv_in,
                             want_state=True)
    assert _scaled(o, o2.view(b, n, H * D).double()) <= 1e-2
    assert _scaled(kv, kv2.double()) <= 1e-5  # same operands, same kernel arithmetic for the state
    assert _scaled(o, _attn64(q, k, v, LAMS, kv_in)) <= 1e-2


@pytest.mark.parametrize("b,n,heads,rot", [(1, 4096, 4, True), (1, 3000, 16, True), (2, 2500, 8, False)])
def test_fused_core_segmented(b, n, heads, rot):
    """batch * heads too small to fill the GPU: the plan splits sequences, and the summary pass applies the
    prologue to kp too -- same result as the two-step path and the fp64 restatement; kv_in / kv_out chain."""
    g = torch.Generator(device=DEV).manual_seed(n)
    qp, kp, v = [(torch.randn(b, n, heads * D, device=DEV, generator=g) * sc).to(torch.bfloat16)
                 for sc in (1.0, 1.0, 0.5)]
    lams = [1.0, 0.999, 0.9, 0.5, 0.05, 0.63, 0.99, 0.3][:heads] + [0.95] * max(0, heads - 8)
    theta = THETA if rot else None
    kv_in = torch.rand(b, heads, D, D, device=DEV) * 0.05
    o, q, k, kv = ops.gla_core_forward(qp, kp, v, lams, heads, theta=theta, offset=3, kv_in=kv_in, want_state=True)
    q2, k2 = ops.gla_prologue(qp, kp, heads, theta=theta, offset=3)
    assert (q - q2).abs().max().item() <= 2 ** -6 * q2.abs().max().item()
    o2, kv2 = ops.la_forward(*(t.view(b, n, heads, D) for t in (q2, k2, v)), lams, layout="bnhd", kv_in=kv_in,
                             want_state=True)
    assert _scaled(o, o2.view(b, n, heads * D).double()) <= 2e-2
    assert _scaled(kv, kv2.double()) <= 2e-2
    # the attention on the kernel's own q / k, against the unsplit fp64 left product
    qh, kh, vh = (t.double().view(b, n, heads, D).transpose(1, 2) for t in (q, k, v))
    lam = torch.tensor(lams, dtype=torch.float64, device=DEV)
    t = torch.arange(n, device=DEV)
    diff = (t[:, None] - t[None, :]).to(torch.float64)
    mask = torch.where(diff[None] >= 0, lam[:, None, None] ** diff.clamp(min=0)[None],
                       torch.zeros((), device=DEV, dtype=torch.float64))
    ref = ((qh @ kh.transpose(-1, -2)) * mask[None]) @ vh
    ref = ref + (lam[None, :, None, None] ** (t.double() + 1)[None, None, :, None]) * (qh @ kv_in.double())
    assert _scaled(o, ref.transpose(1, 2).reshape(b, n, heads * D)) <= 1e-2


def test_fused_core_unsupported_for_fp32():
    qp, kp, v = (t.float() for t in _inputs(6, 256, 3))
    with pytest.raises(UnsupportedError):
        ops.gla_core_forward(qp, kp, v, LAMS, H)


def test_gla_layer_on_the_fused_core_matches_fp64():
    """gla_forward (autograd) with batch * heads = 96 takes the fused forward; y and every gradient within
    the bf16 bars of tests/test_gpu_gla.py (5e-2 / 1.5e-1) of the fp64 restatement."""
    from test_gpu_headline_parity import _gla_reference_fp64

    from paper_2405_17381_b200.gla import GlaWeights, gla_forward

    b, n, dm = 6, 512, H * D
    g = torch.Generator(device=DEV).manual_seed(96)
    rnd = lambda *s, sc=1.0: (torch.randn(*s, device=DEV, generator=g) * sc).to(torch.bfloat16)  # noqa: E731
    x = rnd(b, n, dm, sc=0.5)
    names = ("wq", "wk", "wv", "wu", "wo")
    wbf = {k: rnd(dm, dm, sc=2 * dm ** -0.5) for k in names}
    dy = rnd(b, n, dm, sc=0.5)
    lams = [decay_rate(h, 1, H, 16) for h in range(1, H + 1)]
    xb = x.clone().requires_grad_(True)
    wb = {k: t.clone().requires_grad_(True) for k, t in wbf.items()}
    y = gla_forward(xb, GlaWeights(wb["wq"], wb["wk"], wb["wv"], wb["wo"], wb["wu"]), lams, H, theta=THETA)
    y.backward(dy)
    x64 = x.double().requires_grad_(True)
    w64 = {k: t.double().requires_grad_(True) for k, t in wbf.items()}
    y64 = _gla_reference_fp64(x64, w64, lams, H, THETA)
    y64.backward(dy.double())
    errs = {"y": _scaled(y.detach(), y64.detach()), "dx": _scaled(xb.grad, x64.grad)}
    for k in names:
        errs[f"d{k}"] = _scaled(wb[k].grad, w64[k].grad)
    assert errs["y"] <= 5e-2, errs
    assert all(e <= 1.5e-1 for e in errs.values()), errs


@pytest.mark.parametrize("act,rot,b,n,heads", [("swish", True, 6, 777, 16), ("swish", False, 1, 3000, 4),
                                               ("one_plus_elu", True, 2, 1500, 8), ("none", True, 6, 300, 16)])
def test_fused_core_backward(act, rot, b, n, heads):
    """la_gla_core_bwd: (dqp, dkp, dv) equal the two-step path (la_bwd + la_gla_prologue_bwd) within the bf16
    bar, and the fp64 autograd gradients of the restated core (act, LRPE, decayed attention) within 3e-2 --
    unsplit (batch x heads = 96) and split sequences."""
    g = torch.Generator(device=DEV).manual_seed(n + heads)
    qp, kp, v, da = [(torch.randn(b, n, heads * D, device=DEV, generator=g) * sc).to(torch.bfloat16)
                     for sc in (1.0, 1.0, 0.5, 0.5)]
    lams = ([1.0, 0.999, 0.9, 0.5, 0.05, 0.63, 0.99, 0.3] * 2)[:heads]
    theta = THETA if rot else None
    o, q, k = ops.gla_core_forward(qp, kp, v, lams, heads, act=act, theta=theta, offset=2)
    dqp, dkp, dv = ops.gla_core_backward(qp, kp, q, k, v, da, lams, heads, act=act, theta=theta, offset=2)
    dq2, dk2, dv2 = ops.la_backward(*(t.view(b, n, heads, D) for t in (q, k, v, da)), lams, layout="bnhd")
    dqp2, dkp2, _ = ops.gla_prologue_backward(qp, kp, dq2.view(b, n, -1), dk2.view(b, n, -1), heads, act=act,
                                              theta=theta, offset=2)
    for name, got, ref in (("dqp", dqp, dqp2), ("dkp", dkp, dkp2), ("dv", dv, dv2.view(b, n, -1))):
        assert _scaled(got, ref.double()) <= 2e-2, name
    # fp64 autograd of the restated core on the same bf16 inputs
    qp64, kp64, v64 = (t.double().requires_grad_(True) for t in (qp, kp, v))
    q64, k64 = _act64(qp64, act), _act64(kp64, act)
    if rot:
        q64, k64 = _rot64(q64, THETA, 2), _rot64(k64, THETA, 2)
    qh, kh, vh = (t.view(b, n, heads, D).transpose(1, 2) for t in (q64, k64, v64))
    lam = torch.tensor(lams, dtype=torch.float64, device=DEV)
    t = torch.arange(n, device=DEV)
    diff = (t[:, None] - t[None, :]).to(torch.float64)
    mask = torch.where(diff[None] >= 0, lam[:, None, None] ** diff.clamp(min=0)[None],
                       torch.zeros((), device=DEV, dtype=torch.float64))
    a64 = (((qh @ kh.transpose(-1, -2)) * mask[None]) @ vh).transpose(1, 2).reshape(b, n, heads * D)
    a64.backward(da.double())
    for name, got, ref in (("dqp", dqp, qp64.grad), ("dkp", dkp, kp64.grad), ("dv", dv, v64.grad)):
        assert _scaled(got, ref) <= 3e-2, name
