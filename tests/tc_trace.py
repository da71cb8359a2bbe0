import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops, _lib
lib = _lib.load()
dev = torch.device('cuda', 0)
names = ["tma_issue","S_issued","p_full_ok","O_commit","b_scaled_ok","dS_commit","P_s_full","P_done","O_o_full","O_free","O_store_done","KV_s_full","KV_scaled","KV_ds_full","KV_published","MMA_st_o_ok"]
for (b, n) in ((64, 1024), (8, 8192)):
    q, k, v = (torch.randn(b, 16, n, 128, device=dev, dtype=torch.bfloat16) for _ in range(3))
    lams = [0.99] * 16
    tr = torch.zeros(32 * 16 + 32 * 8 * 4, dtype=torch.int64, device=dev)
    for _ in range(3): ops.la_forward(q, k, v, lams)
    torch.cuda.synchronize()
    lib.la_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    ops.la_forward(q, k, v, lams); torch.cuda.synchronize()
    lib.la_debug_set_trace(ctypes.c_void_p(0))
    t = tr[:512].view(32, 16).cpu().numpy().astype(np.int64)
    tp = tr[512:].view(32, 8, 4).cpu().numpy().astype(np.int64)
    base = t[0, 0]
    print(f"=== b={b} n={n}: cycles relative to chunk0 TMA issue")
    print("chunk " + " ".join(f"{x[:11]:>11s}" for x in names))
    for c in range(32):
        if t[c].max() == 0: break
        print(f"{c:5d} " + " ".join(f"{(x - base) if x else -1:11d}" for x in t[c]))
    print("per P warp (quad, half): [s_full seen, block(half+2) done, A~ done, P done] relative to s_full seen")
    for c in range(4, 8):
        print(f"chunk {c}: " + "  ".join(f"w{w}(q{(w+2)&3},h{w>>2}):{tp[c,w,0]-base}+{tp[c,w,1]-tp[c,w,0]}/{tp[c,w,2]-tp[c,w,0]}/{tp[c,w,3]-tp[c,w,0]}" for w in range(8)))
