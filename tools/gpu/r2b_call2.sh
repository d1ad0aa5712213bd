# Launch floor micro + cfg3 launch list (kernel-only durations under ncu, serialized).
O=gpurun_out/r2b2; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/lf tools/micro/launch_floor.cu && /tmp/lf > $O/launch_floor.txt 2>&1; cat $O/launch_floor.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --workload cfg3_resnet50 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
grep optim8bit $O/launches_cfg3.csv | awk -F'","' '{print $NF}' | tr -d '"' | tail -12
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lars.csv python bench.py --workload lars_resnet50 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
grep -v "^==" $O/launches_lars.csv | awk -F'","' '{print $5, $NF}' | tail -12
