"""CPU oracle for the Lightning Attention hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference package's (``linattn``) ground
truth and its tiled algorithm, so the CUDA path in ``paper_2405_17381_b200``
can be checked on identical inputs.  It is *never* imported by the product
path: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may use it, and there only as the
checker (or as the timed CPU baseline), never as the thing measured or shipped.

Parity status: PINNED.  ``tests/golden/make_golden.py`` runs the real
reference (``/root/reference/pkg/src/linattn``, importable in the build
container) on seeded inputs and commits the outputs under ``tests/golden/``;
``tests/test_oracle.py`` checks every function here against those fixtures and
against the reference test-suite's hand-computed known answers.

Citations are ``file:line`` under ``/root/reference/pkg/src/linattn/``.

Semantics restated
------------------
* decay mask M[t, s] = lam^(t-s) for t >= s, else 0, powers by fp64 cumprod
  (matrixops.py:104-140).
* left product  O = [(Q K^T) * M] V                        (oracles.py:100-115)
* right product kv_t = lam kv_{t-1} + k_t v_t^T, o_t = q_t kv_t (oracles.py:118-131)
* recurrent backward (oracles.py:134-161), left-route backward (oracles.py:164-177)
* tiled forward: per block b of length bl,
      O_b  = [(Q_b K_b^T) * M] V_b + (lam^{1..bl} * Q_b) kv
      kv   = lam^bl kv + (lam^{bl-1..0} * K_b)^T V_b           (kernels.py:253-284)
* tiled backward: sweep 1 rebuilds kv for dQ, sweep 2 (reverse) carries dkv,
  updated *after* block b's dK/dV inter terms                (kernels.py:287-334)
* error metrics max_rel_error / max_scaled_error             (oracles.py:53-81)
* per-head decay lam = exp(-(8h/H)(1 - l/L))                 (positional.py:39-50)

Extensions beyond the reference (needed to check the segment / sequence-
parallel API of the CUDA path): optional ``kv_in`` / ``dkv_in`` initial
states and the final ``kv_out`` / ``dkv_out`` states.  With the defaults
(zeros) the functions reduce exactly to the reference's.
"""

from __future__ import annotations

import math

import numpy as np

REFERENCE = np.float64
WORKING = np.float32
REL_FLOOR = 1e-8  # oracles.py:38


class ShapeError(ValueError):
    """matrixops.py:28-29"""


class DomainError(ValueError):
    """matrixops.py:32-33"""


# --------------------------------------------------------------------------
# substrate: matrixops.py
# --------------------------------------------------------------------------


def check_decay(lam: float) -> float:
    """matrixops.py:72-77 -- lam must lie in (0, 1]."""
    lam = float(lam)
    if not (0.0 < lam <= 1.0):
        raise DomainError(f"decay rate must lie in (0, 1], got {lam}")
    return lam


def decay_powers(count: int, lam: float, first: int = 1) -> np.ndarray:
    """matrixops.py:104-119 -- lam^first .. lam^(first+count-1) by fp64 cumprod."""
    lam = check_decay(lam)
    if count < 0:
        raise DomainError(f"power count must be >= 0, got {count}")
    if count == 0:
        return np.zeros(0, dtype=REFERENCE)
    steps = np.empty(count, dtype=REFERENCE)
    steps[:] = lam
    steps[0] = lam ** first if first else 1.0
    return np.cumprod(steps)


def causal_decay_mask(b: int, lam: float, dtype=REFERENCE) -> np.ndarray:
    """matrixops.py:122-140 -- lower-triangular M[t, s] = lam^(t-s)."""
    if b < 1:
        raise DomainError(f"mask size must be >= 1, got {b}")
    ladder = decay_powers(b, lam, first=0)
    t = np.arange(b)
    diff = t[:, None] - t[None, :]
    out = np.zeros((b, b), dtype=REFERENCE)
    lower = diff >= 0
    out[lower] = ladder[diff[lower]]
    return out.astype(dtype)


def block_count(n: int, B: int) -> tuple[int, int]:
    """matrixops.py:164-171 -- (T, tail) of a length-n sequence cut in B-row blocks."""
    if n < 1 or B < 1:
        raise DomainError(f"need n >= 1 and B >= 1, got n={n}, B={B}")
    T = -(-n // B)
    return T, n - (T - 1) * B


def effective_block(n: int, d: int, B: int | None) -> int:
    """kernels.py:93-97 -- default min(d, n), then clamp into [1, n]."""
    b = min(d, n) if B is None else B
    return max(1, min(b, n))


# --------------------------------------------------------------------------
# metrics: oracles.py:53-81
# --------------------------------------------------------------------------


def max_rel_error(a, b) -> float:
    a = np.asarray(a, dtype=REFERENCE)
    b = np.asarray(b, dtype=REFERENCE)
    if a.shape != b.shape:
        raise ShapeError(f"comparison shapes differ: {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), REL_FLOOR)
    return float((np.abs(a - b) / denom).max())


def max_scaled_error(a, b) -> float:
    a = np.asarray(a, dtype=REFERENCE)
    b = np.asarray(b, dtype=REFERENCE)
    if a.shape != b.shape:
        raise ShapeError(f"comparison shapes differ: {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    scale = max(float(np.abs(a).max()), float(np.abs(b).max()), REL_FLOOR)
    return float(np.abs(a - b).max()) / scale


# --------------------------------------------------------------------------
# ground truth: oracles.py (always float64)
# --------------------------------------------------------------------------


def _as64(*arrays):
    out = [np.asarray(a, dtype=REFERENCE) for a in arrays]
    shape = out[0].shape
    for a in out:
        if a.ndim != 2:
            raise ShapeError(f"expected 2-D input, got ndim={a.ndim}")
        if a.shape != shape:
            raise ShapeError(f"input shapes differ: {shape} vs {a.shape}")
    return out


def left_product_forward(q, k, v, lam: float = 1.0) -> np.ndarray:
    """oracles.py:100-115 -- O(n^2) masked left product."""
    q, k, v = _as64(q, k, v)
    lam = check_decay(lam)
    return ((q @ k.T) * causal_decay_mask(q.shape[0], lam)) @ v


def right_product_forward(q, k, v, lam: float = 1.0, kv_in=None):
    """oracles.py:118-131 -- per-token kv recurrence.  Returns o (and kv_n if kv_in given)."""
    q, k, v = _as64(q, k, v)
    lam = check_decay(lam)
    n, d = q.shape
    kv = np.zeros((d, d)) if kv_in is None else np.array(kv_in, dtype=REFERENCE)
    o = np.empty_like(q)
    for t in range(n):
        kv = lam * kv + np.outer(k[t], v[t])
        o[t] = q[t] @ kv
    return o if kv_in is None else (o, kv)


def reference_backward(q, k, v, do, lam: float = 1.0):
    """oracles.py:134-161 -- closed-form recurrent gradients (dq, dk, dv)."""
    q, k, v, do = _as64(q, k, v, do)
    lam = check_decay(lam)
    n, d = q.shape
    dq, dk, dv = np.empty_like(q), np.empty_like(q), np.empty_like(q)
    kv = np.zeros((d, d))
    for t in range(n):
        kv = lam * kv + np.outer(k[t], v[t])
        dq[t] = do[t] @ kv.T
    dkv = np.zeros((d, d))
    for t in range(n - 1, -1, -1):
        dkv = lam * dkv + np.outer(q[t], do[t])
        dk[t] = v[t] @ dkv.T
        dv[t] = k[t] @ dkv
    return dq, dk, dv


def left_product_backward(q, k, v, do, lam: float = 1.0):
    """oracles.py:164-177 -- gradients through the materialized score matrix."""
    q, k, v, do = _as64(q, k, v, do)
    lam = check_decay(lam)
    m = causal_decay_mask(q.shape[0], lam)
    s = (q @ k.T) * m
    ds = (do @ v.T) * m
    return ds @ k, ds.T @ q, s.T @ do


def finite_difference_grads(f, x, h: float) -> np.ndarray:
    """oracles.py:180-206 -- central differences of scalar f at x, entry by entry."""
    if h <= 0:
        raise ValueError(f"finite-difference step must be > 0, got {h}")
    x = np.array(x, dtype=REFERENCE)
    g = np.empty_like(x)
    for i in range(x.size):
        orig = x.flat[i]
        x.flat[i] = orig + h
        up = f(x)
        x.flat[i] = orig - h
        down = f(x)
        x.flat[i] = orig
        g.flat[i] = (up - down) / (2.0 * h)
    return g


# --------------------------------------------------------------------------
# the tiled algorithm: kernels.py:234-334 (the hot path being replaced)
# --------------------------------------------------------------------------


def _ladders(B: int, lam: float, dt):
    """kernels.py:234-250 -- (mask, lam_out = lam^1..B, pw0 = lam^0..B-1), fp64 then cast."""
    mask = causal_decay_mask(B, lam, dt)
    lam_out = decay_powers(B, lam, first=1).astype(dt)[:, None]
    pw0 = decay_powers(B, lam, first=0)
    return mask, lam_out, pw0


def tiled_forward(q, k, v, lam: float = 1.0, B: int | None = None, dtype=REFERENCE,
                  kv_in=None, return_state: bool = False):
    """kernels.py:253-284 -- blockwise forward in ``dtype``.

    ``kv_in`` (d x d) seeds the carried state (zeros in the reference); with
    ``return_state`` the final state ``kv_n`` is returned as well.
    """
    q, k, v = (np.ascontiguousarray(a, dtype=dtype) for a in (q, k, v))
    n, d = q.shape
    lam = check_decay(lam)
    B = effective_block(n, d, B)
    T, _ = block_count(n, B)
    mask, lam_out, pw0 = _ladders(B, lam, dtype)
    kv = np.zeros((d, d), dtype=dtype) if kv_in is None else np.array(kv_in, dtype=dtype)
    o = np.empty((n, d), dtype=dtype)
    for t in range(T):
        lo, hi = t * B, min(t * B + B, n)
        bl = hi - lo
        qb, kb, vb = q[lo:hi], k[lo:hi], v[lo:hi]
        o[lo:hi] = ((qb @ kb.T) * mask[:bl, :bl]) @ vb + (lam_out[:bl] * qb) @ kv
        lam_in = pw0[:bl][::-1].astype(dtype)[:, None]
        kv = dtype(lam ** bl) * kv + (lam_in * kb).T @ vb
    return (o, kv) if return_state else o


def tiled_backward(q, k, v, do, lam: float = 1.0, B: int | None = None, dtype=REFERENCE,
                   kv_in=None, dkv_in=None, return_state: bool = False):
    """kernels.py:287-334 -- two-sweep blockwise backward in ``dtype``.

    ``kv_in`` seeds sweep 1 (the forward state entering the sequence);
    ``dkv_in`` seeds sweep 2 (the adjoint state arriving from beyond the
    sequence end).  Both are zeros in the reference.  With ``return_state``
    the adjoint state at the sequence start (``dkv_0``) is returned too.
    """
    q, k, v, do = (np.ascontiguousarray(a, dtype=dtype) for a in (q, k, v, do))
    n, d = q.shape
    lam = check_decay(lam)
    B = effective_block(n, d, B)
    T, _ = block_count(n, B)
    mask, lam_out, pw0 = _ladders(B, lam, dtype)
    dq, dk, dv = (np.empty((n, d), dtype=dtype) for _ in range(3))

    kv = np.zeros((d, d), dtype=dtype) if kv_in is None else np.array(kv_in, dtype=dtype)
    for t in range(T):  # sweep 1, kernels.py:309-318
        lo, hi = t * B, min(t * B + B, n)
        bl = hi - lo
        kb, vb, dob = k[lo:hi], v[lo:hi], do[lo:hi]
        dq[lo:hi] = ((dob @ vb.T) * mask[:bl, :bl]) @ kb + (lam_out[:bl] * dob) @ kv.T
        lam_in = pw0[:bl][::-1].astype(dtype)[:, None]
        kv = dtype(lam ** bl) * kv + (lam_in * kb).T @ vb

    dkv = np.zeros((d, d), dtype=dtype) if dkv_in is None else np.array(dkv_in, dtype=dtype)
    for t in range(T - 1, -1, -1):  # sweep 2, kernels.py:320-333
        lo, hi = t * B, min(t * B + B, n)
        bl = hi - lo
        qb, kb, vb, dob = q[lo:hi], k[lo:hi], v[lo:hi], do[lo:hi]
        m = mask[:bl, :bl]
        lam_in = pw0[:bl][::-1].astype(dtype)[:, None]
        dk[lo:hi] = ((dob @ vb.T) * m).T @ qb + (lam_in * vb) @ dkv.T
        dv[lo:hi] = ((qb @ kb.T) * m).T @ dob + (lam_in * kb) @ dkv
        # the adjoint state is updated only after block t used it (kernels.py:331-333)
        dkv = dtype(lam ** bl) * dkv + (lam_out[:bl] * qb).T @ dob
    if return_state:
        return (dq, dk, dv), dkv
    return dq, dk, dv


# --------------------------------------------------------------------------
# decay schedule: positional.py:39-50
# --------------------------------------------------------------------------


def decay_rate(h: int, l: int, H: int, L: int, temperature: bool = True) -> float:
    if not (1 <= h <= H):
        raise DomainError(f"head index {h} outside 1..{H}")
    if not (1 <= l <= L):
        raise DomainError(f"layer index {l} outside 1..{L}")
    scale = (1.0 - l / L) if temperature else 1.0
    return math.exp(-(8.0 * h / H) * scale)


# --------------------------------------------------------------------------
# batched drivers over [batch, heads, n, d] with one lam per head
# (the reference loops over heads in Python: model.py:393-401, 432-442)
# --------------------------------------------------------------------------


def batched_forward(q, k, v, lams, B=None, dtype=REFERENCE, kv_in=None):
    """Returns (o, kv_out) for [b, h, n, d] inputs; kv_in/kv_out are [b, h, d, d]."""
    b, h, n, d = q.shape
    o = np.empty((b, h, n, d), dtype=dtype)
    kv_out = np.empty((b, h, d, d), dtype=dtype)
    for i in range(b):
        for j in range(h):
            o[i, j], kv_out[i, j] = tiled_forward(
                q[i, j], k[i, j], v[i, j], float(lams[j]), B, dtype,
                kv_in=None if kv_in is None else kv_in[i, j], return_state=True)
    return o, kv_out


def batched_backward(q, k, v, do, lams, B=None, dtype=REFERENCE, kv_in=None, dkv_in=None):
    """Returns ((dq, dk, dv), dkv_out) for [b, h, n, d] inputs."""
    b, h, n, d = q.shape
    grads = [np.empty((b, h, n, d), dtype=dtype) for _ in range(3)]
    dkv_out = np.empty((b, h, d, d), dtype=dtype)
    for i in range(b):
        for j in range(h):
            (gq, gk, gv), dkv_out[i, j] = tiled_backward(
                q[i, j], k[i, j], v[i, j], do[i, j], float(lams[j]), B, dtype,
                kv_in=None if kv_in is None else kv_in[i, j],
                dkv_in=None if dkv_in is None else dkv_in[i, j], return_state=True)
            grads[0][i, j], grads[1][i, j], grads[2][i, j] = gq, gk, gv
    return tuple(grads), dkv_out
