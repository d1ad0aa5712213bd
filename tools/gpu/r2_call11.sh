set -x
mkdir -p gpurun_out/r2
for L in 2be13e4 cur; do
AB_ITERS=1 timeout 300 ncu --set full --clock-control none -k regex:optim8bit_step -s 12 -c 1 -o gpurun_out/r2/ab_$L python tools/ab_libs.py tools/ab/libq8_$L.so > /dev/null 2>&1; echo ncu $L $?
done
AB_ITERS=10 timeout 300 python tools/ab_libs.py tools/ab/libq8_cur.so tools/ab/libq8_2be13e4.so; echo ab $?
timeout 900 python -m pytest tests/test_gpu_layerwise.py -q -x -p no:cacheprovider > gpurun_out/r2/pytest_c11.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2/pytest_c11.log
timeout 600 python bench.py --workload lars_resnet50 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench11_lars.json 2> gpurun_out/r2/bench11_lars.err; echo lars $?
tail -c 600 gpurun_out/r2/bench11_lars.json; tail -3 gpurun_out/r2/bench11_lars.err
