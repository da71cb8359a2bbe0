# ncu --set full of the GLA-mode pass kernel (la_gla_core_fwd at [8, 8192, 2048], LRPE on, q / k out)
cat > /tmp/gla_one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2405_17381_b200 import ops
from oracle.linattn_oracle import decay_rate
H, D = 16, 128
lam = [decay_rate(h, 1, H, 16) for h in range(1, H + 1)]
theta = torch.tensor([10000.0 ** (-2.0 * j / D) for j in range(D // 2)], dtype=torch.float64, device="cuda")
qp, kp, v = (torch.randn(8, 8192, H * D, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(3): ops.gla_core_forward(qp, kp, v, lam, H, theta=theta)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_pass_kernel" -s 2 -c 1 -o gpurun_out/r02_gla_full python /tmp/gla_one.py > gpurun_out/ncu_gla.log 2>&1
tail -2 gpurun_out/ncu_gla.log
ncu -i gpurun_out/r02_gla_full.ncu-rep --page raw --csv > gpurun_out/r02_gla_full_raw.csv 2>&1
