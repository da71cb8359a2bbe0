import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops, _lib
lib = _lib.load()
dev = torch.device('cuda', 0)
names = ["tmaA","S_issued","p_full_ok","O_commit","b_scaled_ok","dS_commit","P_s_full","P_done","O_o_full","O_free","O_store_done","KV_s_full","KV_scaled","KV_ds_full","KV_published","MMA_X_issue", "tmaB", "tmaC", "st_issue", "st_read", "S_lands", "-", "MMA_st_rdy", "MMA_ofree"]
shapes = [tuple(map(int, a.split('x'))) for a in sys.argv[1:]] or [(64, 1024), (8, 8192)]
for (b, n) in shapes:
    q, k, v = (torch.randn(b, 16, n, 128, device=dev, dtype=torch.bfloat16) for _ in range(3))
    lams = [0.99] * 16
    tr = torch.zeros(32 * 32 + 32 * 8 * 8, dtype=torch.int64, device=dev)
    for _ in range(3): ops.la_forward(q, k, v, lams)
    torch.cuda.synchronize()
    lib.la_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    ops.la_forward(q, k, v, lams); torch.cuda.synchronize()
    lib.la_debug_set_trace(ctypes.c_void_p(0))
    t = tr[:1024].view(32, 32).cpu().numpy().astype(np.int64)
    tp = tr[1024:].view(32, 8, 8).cpu().numpy().astype(np.int64)
    base = t[0, 0]
    print(f"=== b={b} n={n}: cycles relative to chunk0 TMA issue")
    print("chunk " + " ".join(f"{x[:11]:>11s}" for x in names))
    for c in range(32):
        if t[c].max() == 0: break
        print(f"{c:5d} " + " ".join(f"{(x - base) if x else -1:11d}" for x in t[c][:len(names)]))
    print("per P warp (quad, half), relative to s_full seen: ld1 = block(half+2) TMEM data in, b1 = block done, A~ done, ld2 = block(half) data in, st = P stores issued, P done")
    for c in range(4, 10):
        print(f"chunk {c}:")
        for w in range(8):
            r = tp[c, w] - tp[c, w, 0]
            print(f"   w{w}(q{(w+2)&3},h{w>>2}) @{tp[c,w,0]-base}: ld1 {r[4]} b1 {r[1]} A~ {r[2]} ld2 {r[5]} st {r[6]} done {r[3]}")
