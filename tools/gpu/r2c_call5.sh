# LAMB norms pass as 3 sub-blocks x 256 threads (24 warps/SM) for 16-bit grads: layer-wise parity, ABBA A/B vs 4 x 128.
# (result: 3 x 256 measured 2.7 % slower -- 6822 vs 7009 us over four ABBA pairs -- and dropped)
O=gpurun_out/r2c5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "lamb_gpt2_xl" 20 tools/ab/libq8_new2.so tools/ab/libq8_n3.so 4 > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lamb.csv python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r2c5/launches_lamb.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        if 'q8::' in d['Kernel Name']: print(d['Kernel Name'][:60], d['Metric Value'])
PY
