python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py tests/test_gpu_layerwise.py tests/test_gpu_optim.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/probe_launch.py 2>&1 | grep -E "plan|multi"
for w in cfg3_resnet50 lars_resnet50; do
timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['roofline']['frac'])"
done
