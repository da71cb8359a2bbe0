"""Sequence parallelism across real ranks with the CUDA kernels: 2 and 3 processes share the one GPU of this
run over a ``gloo`` group (NCCL refuses two ranks on one device; the states cross gloo through host copies),
each holding a contiguous slice of every sequence -- both exchanges ("gather": all_gather + decayed prefix /
suffix; "chain": the neighbour P2P chain), uneven slices.  The gathered outputs and gradients must equal the
single-process entry points on the whole sequence (bf16 bar 2e-2, scaled)."""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

B, H, N, D = 1, 4, 2000, 128
LAMS = [1.0, 0.99, 0.9, 0.5]


def _inputs():
    g = torch.Generator().manual_seed(11)
    return [(torch.randn(B, H, N, D, generator=g) * D ** -0.5).to(torch.bfloat16) for _ in range(4)]


def _worker(rank, world, port, cuts, exchange, outdir):
    import torch.distributed as dist

    from paper_2405_17381_b200.sp import sp_lightning_attention

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    q, k, v, do = _inputs()
    lo, hi = cuts[rank], cuts[rank + 1]
    ql, kl, vl = (t[:, :, lo:hi].cuda().requires_grad_(True) for t in (q, k, v))
    o = sp_lightning_attention(ql, kl, vl, LAMS, exchange=exchange)
    o.backward(do[:, :, lo:hi].cuda())
    torch.cuda.synchronize()
    torch.save({"o": o.detach().cpu(), "dq": ql.grad.cpu(), "dk": kl.grad.cpu(), "dv": vl.grad.cpu()},
               os.path.join(outdir, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cuts,exchange", [([0, 1024, 2000], "gather"), ([0, 1024, 2000], "chain"),
                                           ([0, 640, 1280, 2000], "gather"), ([0, 128, 1920, 2000], "chain")])
def test_sequence_parallel_ranks_on_the_cuda_kernels(cuts, exchange, tmp_path):
    from paper_2405_17381_b200 import ops

    world = len(cuts) - 1
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_worker, args=(world, port, cuts, exchange, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    parts = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]
    q, k, v, do = (t.cuda() for t in _inputs())
    want_o = ops.la_forward(q, k, v, LAMS)
    want = dict(zip(("dq", "dk", "dv"), ops.la_backward(q, k, v, do, LAMS)))
    want["o"] = want_o
    for name, ref in want.items():
        got = torch.cat([p[name] for p in parts], dim=2).cuda().float()
        err = ((got - ref.float()).abs().max() / ref.float().abs().max()).item()
        assert err <= 2e-2, (name, err)
