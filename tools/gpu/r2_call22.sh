nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/param_launch tools/micro/param_launch.cu && /tmp/param_launch
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_layerwise.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none -k regex:optim8bit_step -s 3 -c 1 -o gpurun_out/r2/lars2_full python bench.py --workload lars_resnet50 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu $?
