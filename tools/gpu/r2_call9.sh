set -x
mkdir -p gpurun_out/r2
AB_ITERS=5 timeout 300 python tools/ab_libs.py tools/ab/libq8_2be13e4.so tools/ab/libq8_3edcc19.so tools/ab/libq8_cur.so; echo ab $?
for L in 2be13e4 3edcc19 cur; do
AB_ITERS=1 timeout 300 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none -k regex:optim8bit_step -s 12 -c 1 python tools/ab_libs.py tools/ab/libq8_$L.so 2>&1 | grep -E "inst_executed|cycles_elapsed|duration" ; done
