# fp32 tensor-core pass: parity tests, timing vs SIMT, and one ncu --set full capture of the fwd pass kernel
timeout 600 python -m pytest tests/test_gpu_tc32.py -x -q > gpurun_out/tc32_tests.log 2>&1; tail -3 gpurun_out/tc32_tests.log
timeout 300 python tools/tc32_time.py 2>&1 | tail -20
if [ "${TC32_NCU:-0}" = "1" ]; then
  cat > /tmp/tc32_one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2405_17381_b200 import ops
from oracle.linattn_oracle import decay_rate
lams = [decay_rate(h + 1, 1, 16, 16) for h in range(16)]
q, k, v = (torch.randn(8, 16, 8192, 128, device="cuda") / 128 ** 0.5 for _ in range(3))
for _ in range(3): ops.la_forward(q, k, v, lams)
torch.cuda.synchronize()
PY
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc32_pass_kernel" -s 2 -c 1 -o gpurun_out/r02_tc32_full python /tmp/tc32_one.py > gpurun_out/ncu_tc32.log 2>&1
  tail -3 gpurun_out/ncu_tc32.log
  ncu -i gpurun_out/r02_tc32_full.ncu-rep --page raw --csv > gpurun_out/r02_tc32_full_raw.csv 2>&1
fi
