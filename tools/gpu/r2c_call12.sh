# cfg4 step: per-instruction stall attribution (is the per-block absmax load exposed?).
O=gpurun_out/r2c12; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 8 -c 1 -o /tmp/cfg4_full python bench.py --steps 2 --warmup 8 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1; echo ncu $?
ncu -i /tmp/cfg4_full.ncu-rep --page source --csv --print-source sass > $O/cfg4_source.csv 2>/dev/null; echo src $?
python tools/ncu_stalls.py $O/cfg4_source.csv 60 > $O/cfg4_stalls.txt 2>&1; echo st $?
grep -n 'LDG\|LDS.U8\|SYNCS\|BAR' $O/cfg4_stalls.txt | head -30
