# DRAM bytes of the LAMB kernels with the segment build (zero stores) vs the segment-end build (no zero stores).
O=gpurun_out/r2c8; mkdir -p $O
for lib in libq8_seg libq8_new2; do
  Q8_LIB_PATH=tools/ab/$lib.so timeout 600 ncu --metrics dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --csv -k regex:optim8bit_step -s 12 -c 4 --log-file $O/$lib.csv python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo $lib $?
  grep -E 'dram|duration' $O/$lib.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
done
