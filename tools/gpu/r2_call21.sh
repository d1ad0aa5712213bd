python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_optim.py tests/test_gpu_layerwise.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/probe_launch.py
for w in cfg3_resnet50 optim_api_gpt2_xl; do
timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null > gpurun_out/r2/bench21_$w.json; python -c "import json,sys; d=json.loads(open('gpurun_out/r2/bench21_$w.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['roofline']['frac'], d.get('eager'), d.get('cuda_graph'))"
done
