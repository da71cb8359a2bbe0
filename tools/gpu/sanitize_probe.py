# small runs of every kernel for compute-sanitizer (memcheck / racecheck / synccheck): the tcgen05 pass (bf16
# and the fp32 split pass, full and state-only),
# dK/dV sweep, summary and scan kernels (segmented), the SIMT path, decode (bulk and generic), the GLA
# stages (with LRPE) and the TP stages
import sys, torch
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops
for dtype, backend, n, segs in ((torch.bfloat16, "tcgen05", 300, 0), (torch.bfloat16, "tcgen05", 1000, 3),
                                (torch.float32, "simt", 100, 2), (torch.float32, "tcgen05", 300, 0),
                                (torch.float32, "tcgen05", 1000, 3)):
    q, k, v, do = (torch.rand(1, 2, n, 128, device="cuda", dtype=dtype) for _ in range(4))
    o, seg = ops.la_forward(q, k, v, [0.9, 0.99], backend=backend, segments=segs, want_seg_states=True)
    ops.la_backward(q, k, v, do, [0.9, 0.99], backend=backend, segments=segs, fwd_seg_states=seg)
# round 2: short-memory decays (summary CTAs skipped / truncated, scan skips dead slots), long segments with
# sub-segments, strided operands (per-operand TMA maps), the RESUME path, the check flags, PDL chains
for lams in ([0.3, 0.999], [5.5e-4, 0.62]):
    q, k, v, do = (torch.rand(1, 2, 6000, 128, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    o, seg = ops.la_forward(q, k, v, lams, want_seg_states=True)
    ops.la_backward(q, k, v, do, lams, fwd_seg_states=seg)
    ws = ops.new_workspace(tuple(q.shape))
    ops.la_forward_state(k, v, lams, workspace=ws)
    ops.la_forward(q, k, v, lams, workspace=ws, resume=True, check=True)
    ws2 = ops.new_workspace(tuple(q.shape))
    ops.la_backward_state(q, do, lams, workspace=ws2)
    ops.la_backward(q, k, v, do, lams, parts="dkdv", workspace=ws2, resume=True)
    ops.la_backward(q, k, v, do, lams, parts="dq", fwd_seg_states=seg)
qkv = torch.rand(1, 700, 3, 2, 128, device="cuda", dtype=torch.bfloat16)
ops.la_forward(qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2], [0.9, 0.5], layout="bnhd")
ops.la_backward(qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2], qkv[:, :, 0], [0.9, 0.5], layout="bnhd")
for dtype, d in ((torch.bfloat16, 128), (torch.float32, 128), (torch.float64, 64), (torch.float32, 40)):
    q, k, v = (torch.rand(3, 2, d, device="cuda", dtype=dtype) for _ in range(3))
    kv = torch.rand(3, 2, d, d, device="cuda", dtype=ops.state_dtype(dtype))
    ops.la_decode(q, k, v, [0.9, 0.5], kv)
for dtype in (torch.bfloat16, torch.float32):
    qp, kp, a, u, g = (torch.rand(2, 37, 256, device="cuda", dtype=dtype) for _ in range(5))
    theta = torch.rand(32, dtype=torch.float64)
    ops.gla_prologue(qp, kp, 4, theta=theta, offset=5)
    ops.gla_prologue_backward(qp, kp, a, u, 4, theta=theta, offset=5)
    gated, raw = ops.gla_epilogue(a, u, 4)
    ops.gla_epilogue_backward(g, a, u, raw, 4)
    red = torch.zeros(74, 257, device="cuda", dtype=ops.state_dtype(dtype))
    ops.gla_gate_rowsq(a, u, 4, red[:, 256], rowsq_stride=257)
    ops.gla_rowscale(red, 256)
# round 2b: the fused GLA core forward (GLA modes of the pass and summary kernels) and backward (EPI modes),
# unsplit (bh = 96) and split (bh = 4) sequences, LRPE on
theta = torch.rand(64, dtype=torch.float64, device="cuda")
for b, n, h in ((6, 300, 16), (1, 1000, 4)):
    qp, kp, v, da = (torch.rand(b, n, h * 128, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    lam = [0.9, 0.99, 0.5, 1.0] * (h // 4)
    o, q, k = ops.gla_core_forward(qp, kp, v, lam, h, theta=theta, offset=3)
    ops.gla_core_backward(qp, kp, q, k, v, da, lam, h, theta=theta, offset=3)
# round 2c: head dims below 128 on the tensor-core passes (TMA zero fill past d, d x d state masks), with
# entering / exiting states, split sequences and the state-only passes
for dtype in (torch.bfloat16, torch.float32):
    for d in (32, 64, 96):
        q, k, v, do = (torch.rand(1, 2, 1000, d, device="cuda", dtype=dtype) for _ in range(4))
        kv, dkv = (torch.rand(1, 2, d, d, device="cuda") for _ in range(2))
        (o, kvo), seg = ops.la_forward(q, k, v, [0.9, 0.99], backend="tcgen05", segments=3, kv_in=kv,
                                       want_state=True, want_seg_states=True)
        ops.la_backward(q, k, v, do, [0.9, 0.99], backend="tcgen05", segments=3, kv_in=kv, dkv_in=dkv,
                        want_state=True, fwd_seg_states=seg)
        ops.la_forward_state(k, v, [0.9, 0.99], backend="tcgen05", segments=3)
        ops.la_backward_state(q, do, [0.9, 0.99], backend="tcgen05", segments=3)
torch.cuda.synchronize()
print("ok")
