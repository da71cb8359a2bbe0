# sub-segment summaries + L2 prefetch variants
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_pf0.log 2>&1; tail -1 gpurun_out/bench_pf0.log | cut -c1-300
for pf in 2 3 4; do
  LA_B200_LIB=build/var/libpf$pf.so timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_pf$pf.log 2>&1
  tail -1 gpurun_out/bench_pf$pf.log | cut -c1-300
done
