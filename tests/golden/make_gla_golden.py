"""Golden vectors for the GLA layer stages and recurrent decode, from the REAL reference.

Run in the build container, where /root/reference exists:

    python tests/golden/make_gla_golden.py

Writes tests/golden/gla_golden.npz (committed; the GPU box never reads /root/reference).  For
each case it records the reference's ``gla_forward`` output and every gradient of
``gla_backward`` (model.py:365-453) for a random upstream gradient, plus a run of the reference's
per-head decode recurrence (model.py:697-701) through ``decode_step``-equivalent arithmetic on the
same layer (checked here to reproduce the forward's outputs), the summaries after the prefill
and after the last token.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "gla_golden.npz"

# (name, d_model, heads, n, layers, layer, pe_mode, gla_act, gate, seed)
CASES = [
    ("rot_swish_gate", 64, 2, 50, 4, 1, "mix", "swish", True, 11),        # layer 1 of "mix" rotates
    ("norot_swish_gate", 64, 2, 70, 4, 2, "mix", "swish", True, 12),      # layer 2 of "mix" does not
    ("rot_elu_nogate", 96, 3, 33, 2, 1, "lrpe_d", "one_plus_elu", False, 13),
    ("norot_none_gate", 64, 4, 129, 8, 5, "decay_only", "none", True, 14),
]


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    from linattn import model as M  # noqa: E402
    from linattn.positional import apply_lrpe, layer_pe_policy  # noqa: E402

    out = {}
    for name, dm, heads, n, layers, layer, pe, act, gate, seed in CASES:
        cfg = M.ModelConfig(d_model=dm, layers=layers, heads=heads, d_ff=2 * dm, pe_mode=pe, gla_act=act, gate=gate)
        mdl = M.TnlModel.init(cfg, seed=seed)
        # larger weights than the init's 0.02/sqrt(L) so every stage moves the numbers
        rng = np.random.default_rng(seed + 1000)
        w = mdl.blocks[layer - 1].gla
        for nm in ("wq", "wk", "wv", "wu", "wo"):
            getattr(w, nm)[...] = rng.normal(0.0, 1.0 / np.sqrt(dm), (dm, dm))
        x = rng.normal(0.0, 1.0, (n, dm))
        dy = rng.normal(0.0, 1.0, (n, dm))
        rotate = layer_pe_policy(layer, layers, pe) == "lrpe_d"
        lrpe = mdl.lrpe
        y, cache = M.gla_forward(x, w, mdl.schedule, lrpe, layer, cfg)
        grads = {f"g.{nm}": np.zeros_like(getattr(w, nm)) for nm in ("wq", "wk", "wv", "wu", "wo")}
        grads["lrpe.theta"] = np.zeros(cfg.head_dim // 2)
        gr = {f"g.{nm}": grads[f"g.{nm}"] for nm in ("wq", "wk", "wv", "wu", "wo")}
        gr["lrpe.theta"] = grads["lrpe.theta"]
        dx = M.gla_backward(dy, w, lrpe if rotate else None, cfg, cache, gr, "g")
        lam = np.array([mdl.schedule.rate(h + 1, layer) for h in range(heads)])
        # decode: the reference recurrence per head (model.py:684-704) for the GLA layer alone, after a
        # prefill of the first n0 rows
        n0 = n // 2
        dh = cfg.head_dim
        actf, _ = M.ACTIVATIONS[act]
        kv = np.zeros((heads, dh, dh))
        ys_dec = []
        for t in range(n):
            xt = x[t:t + 1]
            q, k = actf(xt @ w.wq), actf(xt @ w.wk)
            v = xt @ w.wv
            u = xt @ w.wu if gate else None
            a = np.empty_like(xt)
            for h in range(heads):
                sl = slice(h * dh, (h + 1) * dh)
                qh, kh = q[:, sl], k[:, sl]
                if rotate:
                    qh, kh = apply_lrpe(qh, lrpe, offset=t), apply_lrpe(kh, lrpe, offset=t)
                kv[h] *= lam[h]
                kv[h] += np.outer(kh[0], v[0, sl])
                a[0, sl] = qh[0] @ kv[h]
            an, _ = M._norm_forward(a, cfg.norm, w.norm.gain, w.norm.bias)
            g = an * u if gate else an
            ys_dec.append((g @ w.wo)[0])
            if t == n0 - 1:
                out[f"{name}.kv_prefill"] = kv.copy()
        y_decode = np.array(ys_dec)
        out[f"{name}.kv_final"] = kv
        out[f"{name}.cfg"] = np.array([dm, heads, n, layers, layer, int(rotate), int(gate), seed, n0])
        out[f"{name}.act"] = np.array(act)
        out[f"{name}.x"] = x
        out[f"{name}.dy"] = dy
        out[f"{name}.lam"] = lam
        out[f"{name}.theta"] = lrpe.theta if lrpe is not None else np.zeros(cfg.head_dim // 2)
        for nm in ("wq", "wk", "wv", "wu", "wo"):
            out[f"{name}.{nm}"] = getattr(w, nm)
            out[f"{name}.d{nm}"] = gr[f"g.{nm}"]
        out[f"{name}.y"] = y
        out[f"{name}.dx"] = dx
        out[f"{name}.dtheta"] = gr["lrpe.theta"]
        # the decode run must reproduce the layer's forward (same arithmetic, recurrent order)
        assert np.max(np.abs(y_decode - y)) < 1e-9 * max(1.0, np.max(np.abs(y))), name
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(CASES)} cases)")


if __name__ == "__main__":
    main()
