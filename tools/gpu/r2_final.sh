# Round-2 final snapshot on one B200 (gpurun): smoke, full GPU suite, every bench workload, launch lists
# and ncu summaries of the kernels changed in session 3 (LARS two-launch form, caller-table quantizer).
set -x
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest $?
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_cfg4_burst.json 2> $O/bench_cfg4_burst.err; echo b1 $?
timeout 900 python bench.py --steps 200 --warmup 10 --no-e2e > $O/bench_cfg4_sustained.json 2> $O/bench_cfg4_sustained.err; echo b2 $?
for w in cfg2_gpt2_medium cfg3_resnet50 codec_gpt2_xl lamb_gpt2_xl lars_resnet50 optim_api_gpt2_xl cfg5_t5_11b; do
  timeout 900 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err; echo $w $?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref $?
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 bench.py --gpus 2 --steps 10 --warmup 3 --workload cfg2_gpt2_medium > $O/bench_shared_w2.json 2> $O/bench_shared_w2.err; echo w2 $?
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29578 bench.py --force-zero1 --zero-fused --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_zero_w1.json 2> $O/bench_zero_w1.err; echo z1 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lars.csv python bench.py --workload lars_resnet50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncull $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 8 -c 1 -o /tmp/cfg4_full python bench.py --steps 2 --warmup 8 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu4 $?
python tools/ncu_metrics.py /tmp/cfg4_full.ncu-rep 1557611200 > $O/ncu_cfg4.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"lars_norms|optim8bit_step" -s 6 -c 2 -o /tmp/lars_full python bench.py --workload lars_resnet50 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncul2 $?
python tools/ncu_metrics.py /tmp/lars_full.ncu-rep > $O/ncu_lars.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:quantize_tma -s 3 -c 2 -o /tmp/codec_full python bench.py --workload codec_gpt2_xl --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncuc $?
python tools/ncu_metrics.py /tmp/codec_full.ncu-rep 1557611200 > $O/ncu_codec.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt
for f in $O/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), d.get('clocks',{}).get('sm_mhz'))" 2>/dev/null; done
