# Exact oracle nearest code + caller-table Markstein: normalizer/parity tests, codec A/B, LAMB norms stalls.
O=gpurun_out/r2b8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_normalizer.py tests/test_gpu_parity.py tests/test_gpu_quantiles.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -3 $O/pytest.log
for rep in 1 2; do for lib in tools/ab/libq8_head.so tools/ab/libq8_new.so; do
  echo -n "$lib "; Q8_LIB_PATH=$lib timeout 300 python bench.py --workload codec_gpt2_xl --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: (round(v['ms'],3), round(v['frac'],3)) for k, v in d['kernels'].items()}, d['dynamic_equals_generic'])"
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 12 -c 1 -o /tmp/lamb_norms python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
ncu -i /tmp/lamb_norms.ncu-rep --page source --csv --print-source sass > $O/lamb_norms_source.csv 2>/dev/null; echo src $?
python tools/ncu_stalls.py $O/lamb_norms_source.csv 40 > $O/lamb_norms_stalls.txt 2>&1; head -50 $O/lamb_norms_stalls.txt
python tools/ncu_metrics.py /tmp/lamb_norms.ncu-rep > $O/ncu_lamb_norms.txt 2>&1; grep -E "==|gpu__time|stalls|inst_exec|issue" $O/ncu_lamb_norms.txt
