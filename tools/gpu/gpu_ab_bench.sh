# same-box A/B of the bench sweep: bash tools/gpu/gpu_ab_bench.sh <reps> <lib> [<lib> ...]
reps=$1; shift
for rep in $(seq $reps); do
for lib in "$@"; do
  LA_B200_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --no-rows --steps 5 > gpurun_out/ab.log 2>&1
  echo "$lib $(tail -1 gpurun_out/ab.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), d['flatness_128k_over_1k'], ' '.join(f\"{n}:{r['fwd_ms']}/{r['bwd_ms']}\" for n,r in d['sweep'].items()))")"
done; done
