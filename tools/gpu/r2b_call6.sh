# Full GPU suite on the committed build; cfg4 kernel source page (per-instruction executed counts).
O=gpurun_out/r2b6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo pytest $?
tail -3 $O/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 8 -c 1 -o /tmp/cfg4_full python bench.py --steps 2 --warmup 8 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu4 $?
ncu -i /tmp/cfg4_full.ncu-rep --page source --csv --print-source sass > $O/cfg4_source.csv 2>/dev/null; echo src $?
python tools/ncu_stalls.py $O/cfg4_source.csv 30 > $O/cfg4_stalls.txt 2>&1; head -5 $O/cfg4_stalls.txt
