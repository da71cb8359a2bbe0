import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import linattn_oracle as orc
from paper_2405_17381_b200 import ops
dev = torch.device('cuda', 0)
def T(a): return torch.tensor(a, device=dev, dtype=torch.bfloat16)
def H(t): return t.double().cpu().numpy()
for (b,h,n) in [(1,1,257),(2,2,257),(1,1,256),(1,1,258),(1,1,385),(2,2,300),(1,2,129),(1,1,1),(1,1,2),(1,1,130)]:
    lams=[1.0,0.9][:h]
    rng=np.random.default_rng(n+b)
    arrs=[rng.uniform(0.05,1.0,(b,h,n,128)) for _ in range(3)]
    t=list(map(T,arrs)); a=list(map(H,t))
    ro,rkv = orc.batched_forward(*a, lams)
    o,kv = ops.la_forward(*t, lams, want_state=True, backend="tcgen05"); torch.cuda.synchronize()
    x=H(o)
    rel=np.abs(x-ro)/np.maximum(np.maximum(np.abs(x),np.abs(ro)),1e-8)
    bad=np.argwhere(rel>0.02)
    rows=sorted(set(map(int,bad[:,2]))) if len(bad) else []
    print(f"b{b} h{h} n{n}: o err {rel.max():.3e} bad entries {len(bad)} rows {rows[:12]} kv err {orc.max_rel_error(H(kv),rkv):.2e}", flush=True)
    if len(bad): 
        i=tuple(bad[0]); print("   first bad", i, x[i], ro[i])
