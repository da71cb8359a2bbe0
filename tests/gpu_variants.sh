# A/B the library variants in build/var against the default build on a short sweep
SL=${SL:-1024,8192,16384,131072}
for lib in paper_2405_17381_b200/libla_b200.so $(ls build/var/lib*.so | grep -v trace); do
  LA_B200_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --seq-lens $SL --steps 5 > gpurun_out/var.log 2>&1
  echo "$lib $(python -c "
import json,sys
d=json.loads(open('gpurun_out/var.log').read().strip().splitlines()[-1])
print(round(d['value']/1e6,2), ' '.join(f\"{n}:{r['fwd_ms']}/{r['bwd_ms']}\" for n,r in d['sweep'].items()))
" 2>&1 | tail -1)"
done
