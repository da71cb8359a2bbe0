export NV_COMPUTE_SANITIZER_MAX_RACECHECK_HAZARDS=100000  # nothing dropped
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/gpu/sanitize_probe.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool: $(grep -E "ERROR SUMMARY|^ok" gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
