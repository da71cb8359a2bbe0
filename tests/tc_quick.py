import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import linattn_oracle as orc
from paper_2405_17381_b200 import ops
dev = torch.device('cuda', 0)
def run(b,h,n,d,lams,rev_check=True, segments=0, dist="pos"):
    rng = np.random.default_rng(n)
    if dist == "pos":
        arrs = [rng.uniform(0.05, 1.0, (b,h,n,d)) for _ in range(4)]
    else:
        arrs = [rng.standard_normal((b,h,n,d))/np.sqrt(d) for _ in range(4)]
    t = [torch.tensor(a, device=dev, dtype=torch.bfloat16) for a in arrs]
    aa = [x.double().cpu().numpy() for x in t]
    o, kv = ops.la_forward(*t[:3], lams, want_state=True, backend="tcgen05", segments=segments)
    torch.cuda.synchronize()
    ro, rkv = orc.batched_forward(*aa[:3], lams)
    metric = orc.max_rel_error if dist == "pos" else orc.max_scaled_error
    e = metric(o.double().cpu().numpy(), ro); ek = metric(kv.double().cpu().numpy(), rkv)
    dq, dk, dv, dkv = ops.la_backward(*t, lams, want_state=True, backend="tcgen05", segments=segments)
    torch.cuda.synchronize()
    (rdq, rdk, rdv), rdkv = orc.batched_backward(*aa, lams)
    eg = [metric(x.double().cpu().numpy(), r) for x, r in zip((dq,dk,dv,dkv),(rdq,rdk,rdv,rdkv))]
    print(f"b={b} h={h} n={n} seg={segments} {dist}: o {e:.3e} kv {ek:.3e} dq/dk/dv/dkv {[f'{x:.3e}' for x in eg]}", flush=True)
run(1,1,128,128,[1.0])
run(1,2,256,128,[0.9,1.0])
run(1,2,300,128,[0.99,0.5])
run(2,3,1000,128,[1.0,0.95,0.6])
run(2,3,1000,128,[1.0,0.95,0.6], segments=3)
run(1,2,640,128,[0.99,0.8], dist="normal")
