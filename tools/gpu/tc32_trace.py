# per-chunk phase trace of the fp32 split pass (LA_TRACE build: tools/build_variant.sh trace -DLA_TRACE,
# run with LA_B200_LIB=build/var/libtrace.so): cycles of thread 0 of CTA (0, 0), relative to the chunk start
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops, _lib
lib = _lib.load()
names = ["start", "go_s", "go_u(B~C)", "B~done", "S_done", "go_x0(P)", "Y+X0_done", "pub1", "A_next", "X1_done", "all_done",
         "O_staged"]
b, n = 8, 8192
q, k, v = (torch.randn(b, 16, n, 128, device="cuda") / 128 ** 0.5 for _ in range(3))
lams = [0.9] * 16
tr = torch.zeros(32 * 16, dtype=torch.int64, device="cuda")
for _ in range(2): ops.la_forward(q, k, v, lams)
torch.cuda.synchronize()
lib.la_debug_set_trace32(ctypes.c_void_p(tr.data_ptr()))
ops.la_forward(q, k, v, lams); torch.cuda.synchronize()
lib.la_debug_set_trace32(ctypes.c_void_p(0))
t = tr.view(32, 16)[:, :12].cpu().numpy().astype(np.int64)
print("chunk period (start to next start):", [int(t[c + 1, 0] - t[c, 0]) for c in range(1, 12)])
print("      " + " ".join(f"{x:>9s}" for x in names))
for c in range(1, 12):
    print(f"{c:5d} " + " ".join(f"{(x - t[c, 0]) if x else -1:9d}" for x in t[c]))
