import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import linattn_oracle as orc
from paper_2405_17381_b200 import ops
dev = torch.device('cuda', 0)
def T(a): return torch.tensor(a, device=dev, dtype=torch.bfloat16)
def H(t): return t.double().cpu().numpy()
def run(b,h,n,lams,segs,dist="pos",reps=3):
    rng = np.random.default_rng(n)
    if dist=="pos": arrs=[rng.uniform(0.05,1.0,(b,h,n,128)) for _ in range(4)]
    else: arrs=[rng.standard_normal((b,h,n,128))/np.sqrt(128) for _ in range(4)]
    t = list(map(T, arrs)); a = list(map(H, t))
    ro,_ = orc.batched_forward(*a[:3], lams); (rq,rk,rv),_ = orc.batched_backward(*a, lams)
    for rep in range(reps):
        o = ops.la_forward(*t[:3], lams, segments=segs, backend="tcgen05")
        g = ops.la_backward(*t, lams, segments=segs, backend="tcgen05"); torch.cuda.synchronize()
        out=[]
        for name,x,r in zip(("o","dq","dk","dv"), (o,)+tuple(g), (ro,rq,rk,rv)):
            x=H(x); bad=np.isnan(x)
            if bad.any():
                idx=np.argwhere(bad.any(-1))
                out.append(f"{name}:NaN rows {len(idx)} first {idx[:4].tolist()}")
            else:
                out.append(f"{name}:{orc.max_scaled_error(x,r):.1e}")
        print(f"b{b} h{h} n{n} lams{lams} segs{segs} rep{rep}: "+" ".join(out), flush=True)
run(1,1,1000,[0.6],1)
run(1,1,1000,[0.6],4)
run(1,1,1000,[1.0],4)
run(1,1,640,[0.8],1)
run(1,1,640,[0.8],2)
run(2,3,1000,[1.0,0.95,0.6],1)
run(2,3,1000,[1.0,0.95,0.6],4)
run(1,2,640,[0.99,0.8],2,dist="normal")
run(1,2,640,[0.99,0.8],1,dist="normal")
