# sustained-load A/B (power-cap regime): tools/step_probe.py 40 steps per arm, alternating, 2 reps.
# Arms are "name:env" pairs, e.g.  bash tools/gpu/gpu_sustained_ab.sh base:LA_PERSISTENT=1 nopers:LA_PERSISTENT=0
# (LA_B200_LIB=<lib> as the env selects a library variant).  Logs: gpurun_out/sp_<name>_<rep>.log
for rep in 1 2; do for arm in "$@"; do
  name=${arm%%:*}; envs=${arm#*:}
  env $envs timeout 300 python tools/step_probe.py 40 > gpurun_out/sp_${name}_$rep.log 2>&1
done; done
