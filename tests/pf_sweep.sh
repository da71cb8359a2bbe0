for pf in 0 2 4 6; do
  LA_B200_LIB=build/var/libla_pf$pf.so timeout 200 python bench.py --no-cpu --no-e2e --seq-lens 1024,8192,131072 --steps 3 > gpurun_out/bench_pf$pf.log 2>&1
done
timeout 200 python bench.py --no-cpu --no-e2e > gpurun_out/bench.log 2>&1
