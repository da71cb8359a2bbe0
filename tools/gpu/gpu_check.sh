# gpu suite + full default bench
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['flatness_128k_over_1k'], d['roofline']['frac'], d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value'))
for n,r in d['sweep'].items(): print(n, r['fwd_ms'], r['bwd_ms'], r['tokens_per_s'])"
