# 40 bench sweeps with nvidia-smi sampled every 20 ms (SM / memory clocks, power, throttle reasons):
# what the board does once it reaches its power cap
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap,temperature.gpu --format=csv,noheader -lms 20 > gpurun_out/power_samples.csv &
SMI=$!
python tools/step_probe.py 40 > gpurun_out/power_steps.txt 2>&1
kill $SMI
tail -5 gpurun_out/power_steps.txt
python - <<'PY'
rows = [l.strip().split(", ") for l in open("gpurun_out/power_samples.csv") if l.strip()]
import statistics
busy = [r for r in rows if float(r[3].split()[0]) > 500]
print("samples", len(rows), "busy", len(busy))
for k in range(0, len(busy), max(1, len(busy) // 12)):
    print(busy[k])
PY
