python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/probe_launch.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:optim8bit_step -s 30 -c 6 python tools/probe_launch.py 2>&1 | grep -E "optim8bit|duration" | head -20
timeout 900 python -m pytest tests/test_gpu_layerwise.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --workload lars_resnet50 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lars', d['ms_per_step'], d['roofline']['frac'])"
