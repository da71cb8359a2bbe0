# sustained A/B of library variants (tools/build_variant.sh <name> [-D...]): per-call la_fwd time burst vs sustained
# (tools/gpu/ko_power.py); STEPS=1 adds 40 bench sweeps per variant (tools/step_probe.py)
# usage: bash tools/gpu/ko_power.sh name1 name2 ...
for rep in 1 2; do for n in "$@"; do LA_B200_LIB=build/var/lib$n.so python tools/gpu/ko_power.py; done; done
[ "${STEPS:-0}" = "1" ] || exit 0
for rep in ${REPS:-1 2}; do for n in "$@"; do
  LA_B200_LIB=build/var/lib$n.so python tools/step_probe.py 40 > gpurun_out/ko_steps_$n.log 2>&1
  python - gpurun_out/ko_steps_$n.log $n <<'PY'
import sys, re
v = [float(re.search(r"total ([0-9.]+)", l).group(1)) for l in open(sys.argv[1]) if l.startswith("step")]
print(f"{sys.argv[2]} sweep: first5 {sum(v[:5]) / 5:.3f} ms, last20 {sum(v[-20:]) / 20:.3f} ms")
PY
done; sleep 3; done
