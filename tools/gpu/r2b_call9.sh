# Caller-table bucket table: normalizer/parity/quantile tests, codec A/B vs HEAD.
O=gpurun_out/r2b9; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_normalizer.py tests/test_gpu_parity.py tests/test_gpu_quantiles.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -3 $O/pytest.log; grep -E "^E " $O/pytest.log | head -5
for rep in 1 2; do for lib in tools/ab/libq8_head.so tools/ab/libq8_new.so; do
  echo -n "$lib "; Q8_LIB_PATH=$lib timeout 300 python bench.py --workload codec_gpt2_xl --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: (round(v['ms'],3), round(v['frac'],3)) for k, v in d['kernels'].items()}, d['dynamic_equals_generic'])"
done; done
