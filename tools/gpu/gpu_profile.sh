# profiling round: launch list of one bench step (cold, serialized), full ncu of the hot kernels
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-rows > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_pass_kernel|tc_dkdv_kernel|tc_summary_kernel" -s 8 -c 4 -o gpurun_out/prof_full python bench.py --seq-lens 16384 --steps 1 --warmup 3 --no-cpu --no-e2e --no-rows > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out | head
