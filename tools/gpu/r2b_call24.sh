# Fused ZeRO kernel (world 1) vs the plain step: device times and ncu instruction split.
O=gpurun_out/r2b24; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/probe_zero.py > $O/probe.txt 2>&1; cat $O/probe.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -c 2 -o /tmp/zero_full python tools/probe_zero.py --ncu > /dev/null 2>&1; echo ncu $?
python tools/ncu_metrics.py /tmp/zero_full.ncu-rep 1557611200 > $O/ncu.txt 2>&1
grep -E "==|gpu__time|instructions per|registers|stalls" $O/ncu.txt
ncu -i /tmp/zero_full.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null; echo src $?
