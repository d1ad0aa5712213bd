python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_cal.so tools/ab/libq8_cur.so tools/ab/libq8_2be13e4.so
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_2be13e4.so tools/ab/libq8_cur.so tools/ab/libq8_cal.so
done 2>&1 | grep -v "\["
timeout 600 ncu --set full --clock-control none -k regex:optim8bit_step -s 3 -c 1 -o /tmp/lars3 python bench.py --workload lars_resnet50 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu $?
python tools/ncu_metrics.py /tmp/lars3.ncu-rep 25557032 | grep -E "gpu__time|dram__bytes|issue_active|stalls"
