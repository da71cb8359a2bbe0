timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "FAILED|Error|assert" | head -8
cat > /tmp/lp.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2405_17381_b200 import ops
from paper_2405_17381_b200.positional import decay_rate
dev = torch.device('cuda', 0)
lams = [decay_rate(h, 1, 16, 16) for h in range(1, 17)]
for b, n in ((4, 16384), (2, 32768), (1, 131072)):
    q, k, v, do = (torch.randn(b, 16, n, 128, device=dev, dtype=torch.bfloat16) * 128 ** -0.5 for _ in range(4))
    for _ in range(2):
        o, seg = ops.la_forward(q, k, v, lams, want_seg_states=True)
        ops.la_backward(q, k, v, do, lams, fwd_seg_states=seg)
    torch.cuda.synchronize()
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers --clock-control none --cache-control none --csv --log-file gpurun_out/lp.csv python /tmp/lp.py > /dev/null 2>&1

