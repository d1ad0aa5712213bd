set -x
mkdir -p gpurun_out/r2
AB_ITERS=10 timeout 300 python tools/ab_libs.py tools/ab/libq8_2be13e4.so tools/ab/libq8_cur.so; echo ab $?
AB_ITERS=1 timeout 300 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none -k regex:optim8bit_step -s 12 -c 1 python tools/ab_libs.py tools/ab/libq8_cur.so 2>&1 | grep -E "inst_executed|cycles_elapsed|duration"
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_gpu_zero_fused.py tests/test_gpu_multirank.py tests/test_gpu_plan.py -q -x -p no:cacheprovider > gpurun_out/r2/pytest_c10.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2/pytest_c10.log
for w in lamb_gpt2_xl cfg3_resnet50; do
timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench10_$w.json 2> gpurun_out/r2/bench10_$w.err; echo $w $?
done
timeout 300 python tools/probe_zero.py; echo probe $?
