python -c "import __graft_entry__ as g; g.build()" > /dev/null
for w in cfg2_gpt2_medium cfg3_resnet50; do
  timeout 600 python bench.py --workload $w --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w $?
done
timeout 900 python bench.py --workload cfg5_t5_11b --no-e2e --steps 50 > gpurun_out/bench_cfg5_t5_11b.json 2> gpurun_out/bench_cfg5_t5_11b.err; echo cfg5 $?
timeout 600 python bench.py --workload lamb_gpt2_xl --steps 100 > gpurun_out/bench_lamb_gpt2_xl.json 2> gpurun_out/bench_lamb.err; echo lamb $?
timeout 600 python bench.py --workload lars_resnet50 --steps 100 > gpurun_out/bench_lars_resnet50.json 2> gpurun_out/bench_lars.err; echo lars $?
for f in gpurun_out/bench_cfg*.json gpurun_out/bench_la*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],4), 'ms', '%.3g'%d['value'], d['roofline']['frac'], d.get('single_tensor_launches'), d['clocks'])"; done
tail -3 gpurun_out/*.err
