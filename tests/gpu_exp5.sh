for v in trbase trpf; do LA_B200_LIB=build/var/lib$v.so timeout 200 python tests/tc_trace_bwd.py 8x8192 > gpurun_out/trace_$v.log 2>&1; done
