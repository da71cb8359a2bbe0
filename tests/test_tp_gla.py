"""Tensor-parallel GLA (paper_2405_17381_b200/tp.py) against the reference layer's golden outputs
(tests/golden/gla_golden.npz; the reference pins gla_parallel_forward == gla_forward,
test_parallel.py:155-234).

* CPU: a real world-size-2 ``gloo`` group; the local stages are a torch / oracle restatement
  (test infrastructure), so what is exercised is the sharding, the single all-reduce of the
  augmented [rows, d_model + 1] partials and the post-reduce row scale.
* GPU: the CUDA stages (la_gla_prologue, la_fwd, la_gla_gate_rowsq, la_gla_rowscale) for P = 1, 2, 4
  shards in one process, the all-reduce replaced by an in-process sum.
"""

import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import linattn_oracle as orc

GOLD = Path(__file__).resolve().parent / "golden" / "gla_golden.npz"
CASES = ["rot_swish_gate", "norot_swish_gate", "rot_elu_nogate", "norot_none_gate"]


def _load(case, dtype=torch.float64, device="cpu"):
    from paper_2405_17381_b200.gla import GlaWeights
    g = np.load(GOLD)
    dm, heads, n, layers, layer, rotate, gate, seed, n0 = (int(x) for x in g[f"{case}.cfg"])
    t = lambda a: torch.tensor(np.asarray(a), dtype=dtype, device=device)  # noqa: E731
    w = GlaWeights(wq=t(g[f"{case}.wq"]), wk=t(g[f"{case}.wk"]), wv=t(g[f"{case}.wv"]), wo=t(g[f"{case}.wo"]),
                   wu=t(g[f"{case}.wu"]) if gate else None)
    theta = torch.tensor(g[f"{case}.theta"], dtype=torch.float64, device=device) if rotate else None
    return dict(x=t(g[f"{case}.x"])[None], w=w, theta=theta, heads=heads, lam=[float(v) for v in g[f"{case}.lam"]],
                act=str(g[f"{case}.act"]), y=g[f"{case}.y"])


class CpuTpOps:
    """torch fp64 / oracle restatement of the four local stages (model.py:57-129, positional.py:126-150)."""

    @staticmethod
    def _act(x, act):
        if act == "swish":
            return x * 0.5 * (1.0 + torch.tanh(0.5 * x))
        if act == "one_plus_elu":
            return torch.where(x > 0, x + 1.0, torch.exp(torch.clamp(x, max=0.0)))
        return x

    def prologue(self, qp, kp, heads, act, theta):
        q, k = self._act(qp, act), self._act(kp, act)
        if theta is not None:
            b, n, w = q.shape
            d = w // heads
            ang = torch.arange(n, dtype=torch.float64)[:, None] * theta[None, :]
            c, s = torch.cos(ang), torch.sin(ang)

            def rot(x):
                x = x.view(b, n, heads, d // 2, 2)
                x1, x2 = x[..., 0], x[..., 1]
                c_, s_ = c[None, :, None, :], s[None, :, None, :]
                return torch.stack((x1 * c_ - x2 * s_, x1 * s_ + x2 * c_), -1).view(b, n, w)
            q, k = rot(q), rot(k)
        return q, k

    def attention(self, q, k, v, lam, heads):
        b, n, w = q.shape
        d = w // heads
        to = lambda x: x.view(b, n, heads, d).permute(0, 2, 1, 3).numpy()  # noqa: E731
        o, _ = orc.batched_forward(to(q), to(k), to(v), list(lam))
        return torch.from_numpy(o).permute(0, 2, 1, 3).reshape(b, n, w)

    def gate_rowsq(self, a, u, heads, rowsq_view, stride):
        rowsq_view.copy_((a * a).sum(-1).reshape(-1))
        return a * u if u is not None else a.clone()

    def rowscale(self, red, out_width, eps):
        r = torch.sqrt(red[:, out_width:])
        return red[:, :out_width] * (out_width ** 0.5) / torch.clamp(r, min=eps)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_17381_b200.tp import gla_tp_forward, shard_gla_weights
        cs = _load(case)
        shard = shard_gla_weights(cs["w"], cs["heads"], world)[rank]
        lam = cs["lam"][shard.head0:shard.head0 + shard.heads]
        y = gla_tp_forward(cs["x"], shard, lam, act=cs["act"], theta=cs["theta"], tp_ops=CpuTpOps())
        result_q.put((rank, y[0].numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["rot_swish_gate", "norot_none_gate"])
def test_tp_two_ranks_gloo_matches_reference_layer(case):
    world = 2
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, result_q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(result_q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _load(case)["y"]
    for r in range(world):  # every rank holds the full output
        assert np.max(np.abs(results[r] - want)) / np.max(np.abs(want)) < 1e-10


def test_shard_gla_weights_restores_and_validates():
    from paper_2405_17381_b200.errors import DomainError
    from paper_2405_17381_b200.tp import shard_gla_weights
    cs = _load("norot_none_gate")
    shards = shard_gla_weights(cs["w"], cs["heads"], 2)
    assert torch.equal(torch.cat([s.weights.wq for s in shards], 1), cs["w"].wq)
    assert torch.equal(torch.cat([s.weights.wo for s in shards], 0), cs["w"].wo)
    assert [s.head0 for s in shards] == [0, cs["heads"] // 2]
    with pytest.raises(DomainError):
        shard_gla_weights(cs["w"], cs["heads"], 3)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("case", CASES)
def test_tp_cuda_stages_match_reference_layer(case, dtype):
    from paper_2405_17381_b200 import ops
    from paper_2405_17381_b200.tp import gla_tp_forward, shard_gla_weights
    dev = torch.device("cuda", 0)
    cs = _load(case, dtype, dev)
    dm = cs["x"].shape[-1]
    tol = {torch.float64: 1e-9, torch.float32: 1e-4}[dtype]
    for world in (1, 2, 4):
        if cs["heads"] % world:
            continue
        partials = []
        for shard in shard_gla_weights(cs["w"], cs["heads"], world):
            lam = cs["lam"][shard.head0:shard.head0 + shard.heads]
            gla_tp_forward(cs["x"], shard, lam, act=cs["act"], theta=cs["theta"], all_reduce=partials.append)
        red = torch.stack(partials).sum(0)  # the all-reduce, in process
        y = ops.gla_rowscale(red, dm).view(1, -1, dm)
        err = float((y[0].double().cpu() - torch.from_numpy(cs["y"])).abs().max() / np.abs(cs["y"]).max())
        assert err <= tol, (world, err)
