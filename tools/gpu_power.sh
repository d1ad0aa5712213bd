# power / clock facts of the box + a per-launch clock trace of the sustained bench
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > gpurun_out/smi_power.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,power.limit,enforced.power.limit,temperature.gpu,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/trace.csv &
PID=$!
python bench.py --no-e2e --no-cpu-baseline --steps 400 > gpurun_out/bench_long.json
kill $PID
python - <<'PY'
rows=[l.strip().split(', ') for l in open('gpurun_out/trace.csv') if l.strip()]
for r in rows[::4]: print(r)
PY
cat gpurun_out/bench_long.json
