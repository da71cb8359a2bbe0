# round-2c profiling of the final library: launch list of one bench step + ncu --set full of the pass kernel and
# the dK/dV sweep at n = 8K (the bench's roofline shape)
set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-rows --no-multi > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_pass_kernel|tc_dkdv_kernel" -s 6 -c 3 -o gpurun_out/r02c_full_8k python bench.py --seq-lens 8192 --steps 1 --warmup 3 --no-cpu --no-e2e --no-rows --no-multi > gpurun_out/ncu_full8k.log 2>&1
python tools/ncu_summary.py gpurun_out/r02c_launches.csv gpurun_out/r02c_full_8k.ncu-rep gpurun_out/r02c > /dev/null 2>&1
ls -la gpurun_out/ | tail -5
