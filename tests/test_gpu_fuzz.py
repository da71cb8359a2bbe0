"""Randomised parity sweep: shapes, dtypes, backends, layouts, forced segment counts, decays and edge
states drawn from a fixed seed, every case checked against the CPU oracle on the same inputs.
LA_FUZZ_CASES=<k> widens the sweep (default 48 cases, a few seconds)."""

import os

import numpy as np
import pytest

from oracle import linattn_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2405_17381_b200 import ops  # noqa: E402

TOL = {torch.float64: 1e-10, torch.float32: 1e-4, torch.bfloat16: 2e-2}
N_CASES = int(os.environ.get("LA_FUZZ_CASES", "48"))


def _case(i):
    rng = np.random.default_rng(9000 + i)
    dtype = [torch.bfloat16, torch.bfloat16, torch.float32, torch.float64][rng.integers(4)]
    d = 128 if dtype == torch.bfloat16 and rng.random() < 0.8 else int(rng.choice([1, 4, 16, 32, 40, 64, 96, 128]))
    if dtype == torch.float64:
        d = min(d, 64)
    b, h = int(rng.integers(1, 4)), int(rng.integers(1, 5))
    n = int(rng.choice([1, 3, 64, 127, 128, 129, 300, 513, 1000, 2048]))
    segments = int(rng.choice([0, 0, 1, 2, 3, 5]))
    layout = "bnhd" if rng.random() < 0.3 else "bhnd"
    lams = [float(rng.choice([1.0, 0.999, 0.99, 0.9, 0.5, 0.05, 5.5e-4])) for _ in range(h)]
    with_kv, with_dkv, saved = rng.random() < 0.5, rng.random() < 0.5, rng.random() < 0.5
    return dict(dtype=dtype, b=b, h=h, n=n, d=d, segments=segments, layout=layout, lams=lams, with_kv=with_kv,
                with_dkv=with_dkv, saved=saved, seed=int(rng.integers(1 << 30)))


def _dev(a, dtype, layout):
    t = torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).to("cuda").to(dtype)
    return t.transpose(1, 2).contiguous() if layout == "bnhd" else t


def _host(t, layout="bhnd"):
    t = t.detach().to(torch.float64)
    if layout == "bnhd":
        t = t.transpose(1, 2)
    return t.cpu().numpy()


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_case(i):
    c = _case(i)
    dtype, b, h, n, d, layout = c["dtype"], c["b"], c["h"], c["n"], c["d"], c["layout"]
    rng = np.random.default_rng(c["seed"])
    q, k, v, do = (rng.uniform(0.05, 1.0, (b, h, n, d)) for _ in range(4))
    kv = rng.uniform(0.0, 0.05, (b, h, d, d)) if c["with_kv"] else None
    dkv = rng.uniform(0.0, 0.05, (b, h, d, d)) if c["with_dkv"] else None
    tq, tk, tv, tdo = (_dev(a, dtype, layout) for a in (q, k, v, do))
    sdt = ops.state_dtype(dtype)
    tkv = None if kv is None else torch.as_tensor(kv, dtype=sdt, device="cuda")
    tdkv = None if dkv is None else torch.as_tensor(dkv, dtype=sdt, device="cuda")
    (o, kv_out), seg = ops.la_forward(tq, tk, tv, c["lams"], kv_in=tkv, want_state=True, layout=layout,
                                    segments=c["segments"], want_seg_states=True)
    dq, dk, dv, dkv_out = ops.la_backward(tq, tk, tv, tdo, c["lams"], kv_in=tkv, dkv_in=tdkv, want_state=True,
                                          layout=layout, segments=c["segments"],
                                          fwd_seg_states=seg if c["saved"] else None)
    # the oracle sees exactly the (rounded) operands the device saw
    qq, kk, vv, dd = (_host(t, layout) for t in (tq, tk, tv, tdo))
    rkvi = None if tkv is None else _host(tkv)
    rdkvi = None if tdkv is None else _host(tdkv)
    ro, rkv = orc.batched_forward(qq, kk, vv, c["lams"], kv_in=rkvi)
    (rdq, rdk, rdv), rdkv = orc.batched_backward(qq, kk, vv, dd, c["lams"], kv_in=rkvi, dkv_in=rdkvi)
    tol = TOL[dtype]
    for name, got, ref in (("o", _host(o, layout), ro), ("kv_out", _host(kv_out), rkv),
                           ("dq", _host(dq, layout), rdq), ("dk", _host(dk, layout), rdk),
                           ("dv", _host(dv, layout), rdv), ("dkv_out", _host(dkv_out), rdkv)):
        err = orc.max_rel_error(got, ref)
        assert err <= tol, f"case {c}: {name} max rel err {err:.3g} > {tol}"
