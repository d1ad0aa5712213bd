# Round-2 session-4 snapshot on one B200: smoke, full GPU suite, every bench workload (cfg4 burst and
# sustained), reference arm, launch list of cfg4, ncu of LAMB (norms pass changed in this session).
set -x
O=gpurun_out/r2cf; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest $?
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_cfg4_burst.json 2> $O/bench_cfg4_burst.err; echo b1 $?
timeout 900 python bench.py --steps 200 --warmup 10 --no-e2e > $O/bench_cfg4_sustained.json 2> $O/bench_cfg4_sustained.err; echo b2 $?
for w in cfg2_gpt2_medium cfg3_resnet50 codec_gpt2_xl lamb_gpt2_xl lars_resnet50 optim_api_gpt2_xl cfg5_t5_11b; do
  timeout 900 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err; echo $w $?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
timeout 900 ncu --set full --clock-control none -k regex:optim8bit_step -s 12 -c 4 -o /tmp/lamb_full python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncula $?
python tools/ncu_metrics.py /tmp/lamb_full.ncu-rep > $O/ncu_lamb.txt 2>&1
python tools/ncu_stalls.py /tmp/lamb_full.ncu-rep > $O/ncu_lamb_stalls.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt
for f in $O/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), d.get('clocks',{}).get('sm_mhz'))" 2>/dev/null; done
