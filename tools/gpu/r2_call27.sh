python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 0 256; do
Q8_LAMB_NORMS_SUBT=$v timeout 600 python bench.py --workload lamb_gpt2_xl --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lamb $v', d['ms_per_step'], d['roofline']['frac'])"
done
Q8_LAMB_NORMS_SUBT=256 timeout 600 python -m pytest tests/test_gpu_layerwise.py -q -x -p no:cacheprovider -k lamb 2>&1 | tail -1
