# LAMB norms pass (after the segment reduction + segment-end scale kernel): ncu --set full of the first
# chunk's norms launch, SASS source page with per-instruction executed counts and stalls.
O=gpurun_out/r2c7; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 12 -c 1 -o /tmp/norms_full python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1; echo ncu $?
python tools/ncu_metrics.py /tmp/norms_full.ncu-rep > $O/ncu_norms.txt 2>&1
ncu -i /tmp/norms_full.ncu-rep --page source --csv --print-source sass > $O/norms_source.csv 2>/dev/null; echo src $?
python tools/ncu_stalls.py $O/norms_source.csv 40 > $O/norms_stalls.txt 2>&1; echo st $?
