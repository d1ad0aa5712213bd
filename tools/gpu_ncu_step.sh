python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 10 -c 1 -o gpurun_out/step_full python tools/probe_step.py --iters 2 > gpurun_out/ncu_step.log 2>&1; echo ncu $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1; echo ncu2 $?
