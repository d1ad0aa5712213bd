# After the 192-entry descriptor tier: plan tests (192 and 450 tensors), smoke, bench lines of cfg3, LARS, cfg4.
O=gpurun_out/r2c16; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_plan.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
for w in cfg3_resnet50 lars_resnet50 optim_api_gpt2_xl; do
  timeout 900 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err; echo $w $?
done
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_cfg4_burst.json 2> $O/bench_cfg4_burst.err; echo b1 $?
for f in $O/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), d.get('clocks',{}))" 2>/dev/null; done
