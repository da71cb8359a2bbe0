timeout 200 python tests/tc_debug4.py > gpurun_out/dbg4.log 2>&1
timeout 200 python tests/tc_debug2.py > gpurun_out/tc_debug2.log 2>&1
timeout 200 python bench.py --no-cpu --no-e2e > gpurun_out/bench.log 2>&1
LA_B200_LIB=build/var/libla_trace.so timeout 120 python tests/tc_trace.py > gpurun_out/trace.log 2>&1
