python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_flatk.so tools/ab/libq8_cur.so tools/ab/libq8_2be13e4.so
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_2be13e4.so tools/ab/libq8_cur.so tools/ab/libq8_flatk.so
done 2>&1 | grep -v "\["
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --workload lars_resnet50 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lars', d['ms_per_step'], d['roofline']['frac'])"
