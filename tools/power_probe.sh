#!/bin/bash
# usage: tools/power_probe.sh "<probe args>"  -> sustained probe (400 iters) with nvidia-smi sampling
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > /tmp/pw.csv &
PID=$!
python tools/probe_step.py $1 --iters 400
kill $PID
python - <<'PY'
import statistics
rows=[l.split(',') for l in open('/tmp/pw.csv') if l.strip()]
sm=[float(r[0]) for r in rows]; pw=[float(r[1]) for r in rows]
busy=[ (s,p) for s,p in zip(sm,pw) if p>300]
print('samples',len(rows),'busy',len(busy),'median sm',statistics.median([b[0] for b in busy]) if busy else None,'median W',statistics.median([b[1] for b in busy]) if busy else None, 'max W', max(pw))
PY
