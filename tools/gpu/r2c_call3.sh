# New LAMB segment tests + LAMB launch list (where the non-kernel ~0.4 ms of a LAMB step goes).
O=gpurun_out/r2c3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layerwise.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lamb.csv python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r2c3/launches_lamb.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['Kernel Name'][:60], d['Metric Value'])
PY
