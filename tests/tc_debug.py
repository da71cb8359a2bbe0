import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import linattn_oracle as orc
from paper_2405_17381_b200 import ops
dev = torch.device('cuda', 0)
rng = np.random.default_rng(0)
def T(a): return torch.tensor(a, device=dev, dtype=torch.bfloat16)
def H(t): return t.double().cpu().numpy()
b,h,n,d = 1,1,512,128
lams=[0.95]
q,k,v,do = [rng.uniform(0.05,1.0,(b,h,n,d)) for _ in range(4)]
tq,tk,tv,tdo = map(T,(q,k,v,do)); qq,kk,vv,dd = map(H,(tq,tk,tv,tdo))
# 1. state-only kernel vs oracle
for segs in (1,2,4):
    kvd = ops.la_forward_state(tk, tv, lams, segments=segs, backend="tcgen05"); torch.cuda.synchronize()
    _, rkv = orc.batched_forward(qq,kk,vv,lams)
    x = H(kvd); print("fwd_state segs", segs, "nan", np.isnan(x).sum(), "err", orc.max_rel_error(np.nan_to_num(x), rkv))
    dkvd = ops.la_backward_state(tq, tdo, lams, segments=segs, backend="tcgen05"); torch.cuda.synchronize()
    (_, _, _), rdkv = orc.batched_backward(qq,kk,vv,dd,lams)
    x = H(dkvd); print("bwd_state segs", segs, "nan", np.isnan(x).sum(), "err", orc.max_rel_error(np.nan_to_num(x), rdkv))
# 2. kv_in single segment
kv0 = rng.uniform(0.0, 0.1, (b,h,d,d))
o = ops.la_forward(tq,tk,tv,lams, kv_in=torch.tensor(kv0, device=dev, dtype=torch.float32), segments=1, backend="tcgen05"); torch.cuda.synchronize()
ro, _ = orc.batched_forward(qq,kk,vv,lams, kv_in=kv0)
x=H(o); print("kv_in seg1 nan rows", np.where(np.isnan(x).any(-1))[-1][:20], "err", orc.max_rel_error(np.nan_to_num(x), ro))
for segs in (1,2,4):
    o = ops.la_forward(tq,tk,tv,lams, segments=segs, backend="tcgen05"); torch.cuda.synchronize()
    ro, _ = orc.batched_forward(qq,kk,vv,lams)
    x=H(o); print("fwd segs", segs, "nan rows", np.where(np.isnan(x).any(-1))[-1][:20], "err", orc.max_rel_error(np.nan_to_num(x), ro))
    g = ops.la_backward(tq,tk,tv,tdo,lams, segments=segs, backend="tcgen05"); torch.cuda.synchronize()
    (rq,rk,rv),_ = orc.batched_backward(qq,kk,vv,dd,lams)
    for name,x,r in zip("qkv", g, (rq,rk,rv)):
        x=H(x); print("  d"+name, "nan rows", np.where(np.isnan(x).any(-1))[-1][:20], "err", orc.max_rel_error(np.nan_to_num(x), r))
