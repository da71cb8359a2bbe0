"""The C ABI is stream-ordered and capture-safe (include/lightning_attn.h): forward, backward (with
sequence segments and the side-stream summaries), decode and the GLA stages replay from a CUDA graph
with the same results as eager calls."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_forward_backward_decode_replay_from_a_cuda_graph():
    from paper_2405_17381_b200 import ops
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    b, h, n, d = 1, 4, 4096, 128  # bh = 4: the plan splits each sequence into segments
    q, k, v, do = (torch.randn(b, h, n, d, device=dev, dtype=torch.bfloat16) * d ** -0.5 for _ in range(4))
    lam = ops.decay_tensor([0.99, 0.9, 0.5, 1.0], h, dev)
    assert ops.segment_count(ops._desc(ops._geometry(q, "bhnd"), q.dtype, None, "auto", 0)) > 1
    qd, kd, vd = (torch.randn(8, h, d, device=dev, dtype=torch.bfloat16) for _ in range(3))
    kv0 = torch.randn(8, h, d, d, device=dev) * 0.01

    def step(kv):
        o, seg = ops.la_forward(q, k, v, None, lam_dev=lam, want_seg_states=True)
        dq, dk, dv = ops.la_backward(q, k, v, do, None, lam_dev=lam, fwd_seg_states=seg)
        od = ops.la_decode(qd, kd, vd, None, kv, lam_dev=lam)
        return o, dq, dk, dv, od

    kv_eager = kv0.clone()
    want = [t.clone() for t in step(kv_eager)]
    kv_graph = kv0.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(kv_graph.clone())  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        got = step(kv_graph)
    g.replay()
    torch.cuda.synchronize()
    for a, w in zip(got, want):
        assert torch.equal(a, w)
    assert torch.equal(kv_graph, kv_eager)


def test_entry_points_from_two_host_threads():
    """Two host threads, each on its own stream, call forward + backward (segmented, with the
    backward's side stream) concurrently: results equal the single-threaded ones."""
    import threading

    from paper_2405_17381_b200 import ops
    dev = torch.device("cuda", 0)
    torch.manual_seed(1)
    shapes = [(1, 4, 4096, 128), (2, 2, 3000, 128)]
    data = [[torch.randn(*s, device=dev, dtype=torch.bfloat16) * 128 ** -0.5 for _ in range(4)] for s in shapes]
    lams = [[0.99, 0.9, 0.5, 1.0], [0.95, 0.7]]

    def run(i):
        q, k, v, do = data[i]
        o, seg = ops.la_forward(q, k, v, lams[i], want_seg_states=True)
        return (o,) + tuple(ops.la_backward(q, k, v, do, lams[i], fwd_seg_states=seg))

    want = [run(0), run(1)]
    torch.cuda.synchronize()
    got, errors = [None, None], []

    def worker(i):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    out = run(i)
                s.synchronize()
            got[i] = out
        except Exception as e:  # noqa: BLE001 -- surfaced below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=120)
    assert not errors, errors
    for i in range(2):
        for a, w in zip(got[i], want[i]):
            assert torch.equal(a, w)


@pytest.mark.parametrize("path", ["fp32_tcgen05", "gla_core"])
def test_round2_paths_replay_from_a_cuda_graph(path):
    """The fp32 split pass (segmented: its state-only summaries, the scan, the three backward passes with the
    side stream) and the fused GLA core forward (segmented: the prologue in the summary pass) replay from a
    CUDA graph bitwise equal to eager calls, and repeated eager calls are bitwise reproducible."""
    from paper_2405_17381_b200 import ops
    dev = torch.device("cuda", 0)
    torch.manual_seed(2)
    h, d = 4, 128
    if path == "fp32_tcgen05":
        q, k, v, do = (torch.randn(1, h, 3000, d, device=dev) * d ** -0.5 for _ in range(4))
        lam = ops.decay_tensor([0.99, 0.9, 0.5, 1.0], h, dev)

        def step():
            o, seg = ops.la_forward(q, k, v, None, lam_dev=lam, want_seg_states=True)
            return (o,) + tuple(ops.la_backward(q, k, v, do, None, lam_dev=lam, fwd_seg_states=seg))
    else:
        qp, kp, vv = (torch.randn(1, 3000, h * d, device=dev).to(torch.bfloat16) for _ in range(3))
        lam = ops.decay_tensor([0.99, 0.9, 0.5, 1.0], h, dev)
        theta = torch.tensor([10000.0 ** (-2.0 * j / d) for j in range(d // 2)], dtype=torch.float64, device=dev)

        def step():
            return ops.gla_core_forward(qp, kp, vv, None, h, theta=theta, lam_dev=lam, offset=7)

    want = [t.clone() for t in step()]
    again = step()
    for a, w in zip(again, want):
        assert torch.equal(a, w)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        got = step()
    g.replay()
    torch.cuda.synchronize()
    for a, w in zip(got, want):
        assert torch.equal(a, w)
