# one GPU round-trip: correctness probes, full gpu suite, bench, trace
timeout 200 python tests/tc_debug2.py > gpurun_out/tc_debug2.log 2>&1
echo "nan lines: $(grep -c NaN gpurun_out/tc_debug2.log)" >> gpurun_out/summary.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench.log 2>&1
LA_B200_LIB=build/var/libla_trace.so timeout 120 python tests/tc_trace.py > gpurun_out/trace.log 2>&1
cat gpurun_out/summary.txt
