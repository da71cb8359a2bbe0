timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do
for lib in paper_2405_17381_b200/libla_b200.so $(ls build/var/lib*.so | grep -v trace); do echo "$lib $(LA_B200_LIB=$lib timeout 120 python tools/exp_time.py 2>&1 | tail -1)"; done
done
LA_B200_LIB=build/var/libla_trace.so timeout 200 python tools/gpu/tc_trace_bwd.py 8x8192 > gpurun_out/trace_bwd.log 2>&1
