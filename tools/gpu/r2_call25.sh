python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_rul0.so tools/ab/libq8_rul10.so tools/ab/libq8_cur.so tools/ab/libq8_2be13e4.so
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_2be13e4.so tools/ab/libq8_cur.so tools/ab/libq8_rul10.so tools/ab/libq8_rul0.so
done 2>&1 | grep -v "\["
timeout 300 python tools/probe_zero.py
timeout 600 python -m pytest tests/test_gpu_zero_fused.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider 2>&1 | tail -2
