"""The NCCL plumbing on the GPU box: sequence-parallel attention and the TP GLA layer through a real
``nccl`` process group of one rank (this run has one GPU; the multi-rank host logic is covered by the
world-size-2 ``gloo`` tests).  With one rank the exchange is trivial, so each result must equal the
single-GPU entry point it decomposes."""

import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2405_17381_b200 import gla, ops  # noqa: E402


@pytest.fixture(scope="module")
def nccl_group():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_sequence_parallel_over_nccl(nccl_group):
    from paper_2405_17381_b200.sp import sp_lightning_attention
    torch.manual_seed(3)
    b, h, n, d = 2, 4, 1536, 128
    lams = [1.0, 0.99, 0.9, 0.5]
    q, k, v, do = (torch.randn(b, h, n, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5 for _ in range(4))
    ql, kl, vl = (t.clone().requires_grad_(True) for t in (q, k, v))
    o = sp_lightning_attention(ql, kl, vl, lams, group=nccl_group)
    o.backward(do)
    want_o = ops.la_forward(q, k, v, lams)
    want = ops.la_backward(q, k, v, do, lams)
    for got, ref in ((o, want_o), (ql.grad, want[0]), (kl.grad, want[1]), (vl.grad, want[2])):
        err = ((got.float() - ref.float()).abs().max() / ref.float().abs().max()).item()
        assert err <= 2e-2, err


def test_tensor_parallel_gla_over_nccl(nccl_group):
    from paper_2405_17381_b200.tp import gla_tp_forward, shard_gla_weights
    torch.manual_seed(4)
    b, n, heads, d = 2, 300, 4, 64
    dm = heads * d
    x = torch.randn(b, n, dm, device="cuda", dtype=torch.float32)
    w = gla.GlaWeights(*(torch.randn(dm, dm, device="cuda") * dm ** -0.5 for _ in range(5)))
    lams = [0.99, 0.9, 0.7, 0.5]
    theta = torch.rand(d // 2, dtype=torch.float64) * 0.1
    shard = shard_gla_weights(w, heads, 1)[0]
    lam_dev = ops.decay_tensor(lams, heads, x.device)
    y = gla_tp_forward(x, shard, lam_dev, group=nccl_group, theta=theta)
    want = gla.gla_forward(x, w, lams, heads, theta=theta)
    err = ((y - want).abs().max() / want.abs().max()).item()
    assert err <= 1e-4, err
