"""Sequence-parallel host logic (paper_2405_17381_b200/sp.py) under a real
world-size-2 ``gloo`` process group on CPU.

The local kernels are the CPU oracle (test infrastructure) plugged in through
the ``LocalKernels`` interface, so what is exercised here is exactly the
multi-rank part: the summary all_gather, the decayed prefix/suffix combine,
the kv_in / dkv_in hand-off, and the autograd wiring.  Ground truth is the
oracle on the whole, unsplit sequence.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import linattn_oracle as orc


class OracleKernels:
    """LocalKernels on the CPU oracle (fp64), [b, h, n, d] tensors."""

    @staticmethod
    def _np(t):
        return t.detach().to(torch.float64).numpy()

    def forward_state(self, k, v, lam):
        lams = lam.tolist()
        z = np.zeros_like(self._np(k))
        _, kv = orc.batched_forward(z, self._np(k), self._np(v), lams)
        return torch.from_numpy(kv), None

    def forward(self, q, k, v, lam, kv_in, ctx):
        o, _ = orc.batched_forward(self._np(q), self._np(k), self._np(v), lam.tolist(),
                                   kv_in=self._np(kv_in))
        return torch.from_numpy(o), None

    def backward_state(self, q, do, lam):
        lams = lam.tolist()
        z = np.zeros_like(self._np(q))
        _, dkv = orc.batched_backward(self._np(q), z, z, self._np(do), lams)
        return torch.from_numpy(dkv), None

    def begin_dq(self, q, k, v, do, lam, kv_in, seg):
        (dq, _, _), _ = orc.batched_backward(self._np(q), self._np(k), self._np(v), self._np(do), lam.tolist(),
                                             kv_in=self._np(kv_in))
        return torch.from_numpy(dq)

    def backward_dkdv(self, q, k, v, do, lam, dkv_in, ctx):
        (_, dk, dv), _ = orc.batched_backward(self._np(q), self._np(k), self._np(v), self._np(do), lam.tolist(),
                                              dkv_in=self._np(dkv_in))
        return torch.from_numpy(dk), torch.from_numpy(dv)

    def finish_dq(self, handle):
        return handle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cuts, q, k, v, do, lams, result_q, exchange="gather"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_17381_b200.sp import sp_lightning_attention

        lo, hi = cuts[rank], cuts[rank + 1]
        sl = lambda x: x[:, :, lo:hi].clone().requires_grad_(True)  # noqa: E731
        ql, kl, vl = sl(q), sl(k), sl(v)
        lam = torch.tensor(lams, dtype=torch.float64)
        # the last cut pattern passes the slice lengths (no lengths exchange); the others exchange them
        known = [cuts[i + 1] - cuts[i] for i in range(world)] if cuts in ((0, 1, 50), (0, 20, 21, 60)) else None
        o = sp_lightning_attention(ql, kl, vl, lam, kernels=OracleKernels(), lengths=known, exchange=exchange)
        o.backward(do[:, :, lo:hi])
        result_q.put((rank, o.detach().numpy(), ql.grad.numpy(), kl.grad.numpy(), vl.grad.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["gather", "chain"])
@pytest.mark.parametrize("cuts", [(0, 48, 96), (0, 37, 97), (0, 1, 50), (0, 20, 21, 60)])
def test_sequence_parallel_ranks_match_whole_sequence(cuts, exchange):
    """World size 2 (and 3 for the 4-cut pattern, with a one-position middle slice) under gloo: the
    all_gather combine and the P2P neighbour chain both reproduce the unsplit sequence."""
    rng = np.random.default_rng(sum(cuts))
    b, h, d = 2, 3, 8
    n = cuts[-1]
    lams = [1.0, 0.95, 0.6]
    q, k, v, do = (torch.from_numpy(rng.uniform(0.05, 1.0, (b, h, n, d))) for _ in range(4))
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    world = len(cuts) - 1
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cuts, q, k, v, do, lams, result_q, exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict((r[0], r[1:]) for r in (result_q.get(timeout=240) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_o, _ = orc.batched_forward(q.numpy(), k.numpy(), v.numpy(), lams)
    (rdq, rdk, rdv), _ = orc.batched_backward(q.numpy(), k.numpy(), v.numpy(), do.numpy(), lams)
    o = np.concatenate([results[r][0] for r in range(world)], axis=2)
    grads = [np.concatenate([results[r][i] for r in range(world)], axis=2) for i in (1, 2, 3)]
    assert orc.max_rel_error(o, ref_o) < 1e-10
    for g, ref in zip(grads, (rdq, rdk, rdv)):
        assert orc.max_rel_error(g, ref) < 1e-10


def test_prefix_and_suffix_combine_order():
    """The decayed prefix/suffix combine equals the serial state recurrence over 4 slices."""
    from paper_2405_17381_b200.sp import prefix_states, suffix_states

    rng = np.random.default_rng(3)
    b, h, d = 1, 2, 4
    lengths = [5, 1, 7, 3]
    lam = torch.tensor([0.9, 0.5], dtype=torch.float64)
    ks = [rng.uniform(0.05, 1.0, (b, h, n, d)) for n in lengths]
    vs = [rng.uniform(0.05, 1.0, (b, h, n, d)) for n in lengths]
    deltas = [torch.from_numpy(orc.batched_forward(np.zeros_like(kk), kk, vv, lam.tolist())[1])
              for kk, vv in zip(ks, vs)]
    full_k, full_v = np.concatenate(ks, axis=2), np.concatenate(vs, axis=2)
    for p in range(len(lengths)):
        upto = sum(lengths[:p])
        want = orc.batched_forward(np.zeros_like(full_k[:, :, :upto]) if upto else np.zeros((b, h, 1, d)),
                                   full_k[:, :, :upto] if upto else np.zeros((b, h, 1, d)),
                                   full_v[:, :, :upto] if upto else np.zeros((b, h, 1, d)), lam.tolist())[1]
        got = prefix_states(deltas, lengths, lam, p).numpy()
        assert np.allclose(got, want, rtol=1e-12, atol=1e-14)
    qs = [rng.uniform(0.05, 1.0, (b, h, n, d)) for n in lengths]
    dos = [rng.uniform(0.05, 1.0, (b, h, n, d)) for n in lengths]
    rs = [torch.from_numpy(orc.batched_backward(qq, np.zeros_like(qq), np.zeros_like(qq), dd, lam.tolist())[1])
          for qq, dd in zip(qs, dos)]
    full_q, full_do = np.concatenate(qs, axis=2), np.concatenate(dos, axis=2)
    for p in range(len(lengths)):
        start = sum(lengths[:p + 1])
        if start == sum(lengths):
            want = np.zeros((b, h, d, d))
        else:
            tail_q, tail_do = full_q[:, :, start:], full_do[:, :, start:]
            want = orc.batched_backward(tail_q, np.zeros_like(tail_q), np.zeros_like(tail_q), tail_do,
                                        lam.tolist())[1]
        got = suffix_states(rs, lengths, lam, p).numpy()
        assert np.allclose(got, want, rtol=1e-12, atol=1e-14)
