set -x
timeout 200 python tests/tc_debug2.py > gpurun_out/dbg_ahead.log 2>&1
LA_B200_LIB=build/var/libla_noahead.so timeout 200 python tests/tc_debug2.py > gpurun_out/dbg_noahead.log 2>&1
grep -c NaN gpurun_out/dbg_ahead.log gpurun_out/dbg_noahead.log
