set -x
for r in 1 2; do
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_cur.so tools/ab/libq8_late.so tools/ab/libq8_2be13e4.so
AB_ITERS=20 timeout 300 python tools/ab_libs.py tools/ab/libq8_2be13e4.so tools/ab/libq8_late.so tools/ab/libq8_cur.so
done
