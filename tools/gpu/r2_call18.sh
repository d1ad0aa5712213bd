set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in cfg3_resnet50 lars_resnet50 lamb_gpt2_xl; do
timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench18_$w.json 2> gpurun_out/r2/bench18_$w.err; echo $w $?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 12 -c 4 -o /tmp/lamb_full python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_lamb.log 2>&1; echo ncul $?
python tools/ncu_metrics.py /tmp/lamb_full.ncu-rep > gpurun_out/r2/ncu_lamb_sum.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 3 -c 1 -o gpurun_out/r2/lars_full python bench.py --workload lars_resnet50 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_lars.log 2>&1; echo ncur $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 4 -c 1 -o gpurun_out/r2/cfg3b_full python bench.py --workload cfg3_resnet50 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_cfg3b.log 2>&1; echo ncu3 $?
ls -la gpurun_out/r2/*.ncu-rep
