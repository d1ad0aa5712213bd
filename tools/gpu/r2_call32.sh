python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/r2
for w in cfg3_resnet50 lars_resnet50; do
timeout 600 python bench.py --workload $w --steps 50 --warmup 5 > gpurun_out/r2/bench32_$w.json 2>/dev/null; python -c "import json,sys; d=json.loads(open('gpurun_out/r2/bench32_$w.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['roofline']['frac'], d.get('single_tensor_launches'))"
done
