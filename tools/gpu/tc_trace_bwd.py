"""Per-chunk event trace of the fused dK/dV sweep (LA_TRACE build): LA_B200_LIB=build/var/libla_trace.so"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops, _lib
lib = _lib.load()
dev = torch.device('cuda', 0)
names = ["tmaQ", "tmaD", "tmaK", "tmaV", "Sv", "Sk", "st_iss", "dV_iss", "dV_com", "dK_iss", "dK_com", "PvS", "PvE",
         "PkS", "PkE", "W_rdy", "epiV", "epiK", "ST_ds", "ST_pub", "stV", "stRd", "Kfull", "ovf", "Qfull"]
shapes = [tuple(map(int, a.split('x'))) for a in sys.argv[1:]] or [(8, 8192)]
for (b, n) in shapes:
    q, k, v, do = (torch.randn(b, 16, n, 128, device=dev, dtype=torch.bfloat16) * 128 ** -0.5 for _ in range(4))
    lams = [0.99] * 16
    tr = torch.zeros(32 * 32, dtype=torch.int64, device=dev)
    for _ in range(3): ops.la_backward(q, k, v, do, lams)
    torch.cuda.synchronize()
    lib.la_debug_set_trace_bwd_c(ctypes.c_void_p(tr.data_ptr()))
    ops.la_backward(q, k, v, do, lams); torch.cuda.synchronize()
    lib.la_debug_set_trace_bwd_c(ctypes.c_void_p(0))
    t = tr.view(32, 32).cpu().numpy().astype(np.int64)[:, :len(names)]
    print(f"=== b={b} n={n}: cycles relative to each chunk's Sv issue")
    print("chunk " + " ".join(f"{x:>6s}" for x in names) + " period")
    for c in range(2, 20):
        if t[c].max() == 0: break
        base = t[c, 4]
        print(f"{c:5d} " + " ".join(f"{(x - base) if x else -1:6d}" for x in t[c]) + f" {base - t[c-1, 4]:6d}")
