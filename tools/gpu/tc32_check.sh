# fp32 tensor-core pass: parity tests, then timing vs SIMT
timeout 600 python -m pytest tests/test_gpu_tc32.py -x -q > gpurun_out/tc32_tests.log 2>&1; tail -25 gpurun_out/tc32_tests.log
timeout 300 python tools/tc32_time.py 2>&1 | tail -20
