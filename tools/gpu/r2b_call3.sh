# Staged tails: parity of every multi-tensor path, then cfg3 / LARS / LAMB lines and the cfg3 launch list.
O=gpurun_out/r2b3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py tests/test_gpu_layerwise.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo pytest $?
tail -3 $O/pytest.log
for w in cfg3_resnet50 lars_resnet50 lamb_gpt2_xl; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo $w $?
  python -c "import json,sys; d=json.load(open('$O/bench_$w.json')); print('$w', d['ms_per_step'], d['roofline']['frac'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --workload cfg3_resnet50 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
grep -v "^==" $O/launches_cfg3.csv | grep optim8bit | awk -F'","' '{print $5, $NF}' | head -8
