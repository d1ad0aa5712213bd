# Round-2 end state (HEAD after session 4): smoke, full GPU suite, default bench line, every workload,
# reference arm, cfg4 launch list.
O=gpurun_out/r2cf2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest $?
tail -2 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_cfg4_burst.json 2> $O/bench_cfg4_burst.err; echo b1 $?
timeout 900 python bench.py --steps 200 --warmup 10 --no-e2e > $O/bench_cfg4_sustained.json 2> $O/bench_cfg4_sustained.err; echo b2 $?
for w in cfg2_gpt2_medium cfg3_resnet50 lamb_gpt2_xl lars_resnet50 cfg5_t5_11b; do
  timeout 900 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err; echo $w $?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
for f in $O/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), d.get('clocks',{}))" 2>/dev/null; done
