"""Pin the CPU oracle (oracle/linattn_oracle.py) to the real reference.

Every check compares the oracle with outputs the reference package itself
produced (tests/golden/golden.npz, made by tests/golden/make_golden.py) or
with the reference test-suite's hand-computed known answers.  CPU only.
"""

import numpy as np
import pytest

from conftest import case_inputs, config1_inputs, golden, golden_array, golden_cases, golden_config1
from oracle import linattn_oracle as orc

CASES = golden_cases()


def test_hand_case_forward():
    # test_kernels.py:39-54 / test_oracles.py:20-31
    q = k = np.array([[1.0], [1.0]])
    v = np.array([[1.0], [2.0]])
    for B in (1, 2):
        assert np.array_equal(orc.tiled_forward(q, k, v, 1.0, B), [[1.0], [3.0]])
        assert np.allclose(orc.tiled_forward(q, k, v, 0.5, B), [[1.0], [2.5]], rtol=0, atol=1e-15)
    assert np.array_equal(orc.left_product_forward(q, k, v, 0.5), [[1.0], [2.5]])


def test_single_token_backward():
    # test_kernels.py:120-123: (dq, dk, dv) = (15, 10, 6)
    g = orc.tiled_backward(np.array([[2.0]]), np.array([[3.0]]), np.array([[5.0]]), np.array([[1.0]]))
    assert tuple(float(x.item()) for x in g) == (15.0, 10.0, 6.0)


def test_zero_cotangent():
    # test_kernels.py:113-117
    q, k, v = case_inputs(10, 4, 6, "pos", 3)
    for part in orc.tiled_backward(q, k, v, np.zeros((10, 4)), 0.7, 4):
        assert np.array_equal(part, np.zeros((10, 4)))


def test_substrate_known_answers():
    g = golden()
    assert np.array_equal(orc.causal_decay_mask(7, 0.6), g["substrate/mask_7_0.6"])
    assert np.array_equal(orc.decay_powers(9, 0.7, 1), g["substrate/powers_9_0.7_first1"])
    assert np.array_equal(orc.decay_powers(9, 0.7, 0), g["substrate/powers_9_0.7_first0"])
    table = np.array([[orc.decay_rate(h, l, 16, 16) for l in range(1, 17)] for h in range(1, 17)])
    assert np.array_equal(table, g["substrate/decay_rate_H16_L16"])
    # test_matrixops.py:107-113: binary mask at lam=1
    assert np.array_equal(orc.causal_decay_mask(9, 1.0), np.tril(np.ones((9, 9))))


def test_errors():
    with pytest.raises(orc.DomainError):
        orc.check_decay(1.5)
    with pytest.raises(orc.DomainError):
        orc.check_decay(0.0)
    with pytest.raises(orc.ShapeError):
        orc.max_rel_error(np.ones(3), np.ones(4))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference_outputs(case):
    name, n, d, B, lam, seed, dist = case
    q, k, v, do = case_inputs(n, d, seed, dist)
    o64 = orc.tiled_forward(q, k, v, lam, B)
    dq64, dk64, dv64 = orc.tiled_backward(q, k, v, do, lam, B)
    o32 = orc.tiled_forward(q, k, v, lam, B, dtype=np.float32)
    dq32, dk32, dv32 = orc.tiled_backward(q, k, v, do, lam, B, dtype=np.float32)
    for key, got, tol in (("o64", o64, 1e-12), ("dq64", dq64, 1e-12), ("dk64", dk64, 1e-12),
                          ("dv64", dv64, 1e-12), ("o32", o32, 1e-5), ("dq32", dq32, 1e-5),
                          ("dk32", dk32, 1e-5), ("dv32", dv32, 1e-5)):
        ref, view = golden_array(f"{name}/{key}", got)
        metric = orc.max_rel_error if dist == "pos" else orc.max_scaled_error
        assert metric(view(got), ref) <= tol, f"{name}/{key}"
    if f"{name}/left" in golden():
        g = golden()
        assert orc.max_scaled_error(orc.left_product_forward(q, k, v, lam), g[f"{name}/left"]) < 1e-13
        for got, key in zip(orc.reference_backward(q, k, v, do, lam), ("rdq", "rdk", "rdv")):
            assert orc.max_scaled_error(got, g[f"{name}/{key}"]) < 1e-13
        for got, key in zip(orc.left_product_backward(q, k, v, do, lam), ("rdq", "rdk", "rdv")):
            assert orc.max_scaled_error(got, g[f"{name}/{key}"]) < 1e-10


def test_config1_against_reference():
    c = golden_config1()
    q, k, v, do = config1_inputs()
    g = golden()
    for h, lam in enumerate(c["lams"]):
        for dt, tag, tol in ((np.float64, "64", 1e-12), (np.float32, "32", 1e-5)):
            o = orc.tiled_forward(q[0, h], k[0, h], v[0, h], lam, c["B"], dtype=dt)
            grads = orc.tiled_backward(q[0, h], k[0, h], v[0, h], do[0, h], lam, c["B"], dtype=dt)
            for key, arr in zip(("o", "dq", "dk", "dv"), (o,) + tuple(grads)):
                ref, view = golden_array(f"config1/h{h}/{key}{tag}", arr)
                assert orc.max_rel_error(view(arr), ref) <= tol, (h, key, tag)


@pytest.mark.parametrize("lam", [1.0, 0.9, 0.5])
def test_state_extension_composes(lam):
    """kv_out / kv_in (our extension) chains segments exactly (right-product kv)."""
    q, k, v, do = case_inputs(37, 5, 3, "pos")
    whole = orc.tiled_forward(q, k, v, lam, 4)
    o1, kv1 = orc.tiled_forward(q[:16], k[:16], v[:16], lam, 4, return_state=True)
    o2 = orc.tiled_forward(q[16:], k[16:], v[16:], lam, 4, kv_in=kv1)
    assert orc.max_rel_error(np.vstack([o1, o2]), whole) < 1e-12
    _, kv_n = orc.right_product_forward(q, k, v, lam, kv_in=np.zeros((5, 5)))
    _, kv_t = orc.tiled_forward(q, k, v, lam, 7, return_state=True)  # ragged tail 37 = 5*7+2
    assert orc.max_rel_error(kv_t, kv_n) < 1e-12
    # backward: right segment first (it produces the adjoint state entering the left one)
    g_whole = orc.tiled_backward(q, k, v, do, lam, 4)
    _, kv_mid = orc.tiled_forward(q[:16], k[:16], v[:16], lam, 4, return_state=True)
    g2, dkv_mid = orc.tiled_backward(q[16:], k[16:], v[16:], do[16:], lam, 4, kv_in=kv_mid, return_state=True)
    g1 = orc.tiled_backward(q[:16], k[:16], v[:16], do[:16], lam, 4, dkv_in=dkv_mid)
    for a, b, w in zip(g1, g2, g_whole):
        assert orc.max_rel_error(np.vstack([a, b]), w) < 1e-12
