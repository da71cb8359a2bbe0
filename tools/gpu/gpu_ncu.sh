# ncu --set full of the fwd pass kernel and the fused dK/dV kernel at n=8192 (one launch each)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_pass_kernel|tc_dkdv_kernel" -s 6 -c 3 -o gpurun_out/prof_full python bench.py --seq-lens 8192 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/prof_full_raw.csv 2>&1
ls -la gpurun_out/
