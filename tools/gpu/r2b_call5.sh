# LARS (contiguous-range norms + scales, PDL step) parity + A/B; cfg3 kernel source-level stalls.
O=gpurun_out/r2b5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo pytest $?
tail -3 $O/pytest.log
bash tools/ab_work.sh "lars_resnet50" 30 tools/ab/libq8_head.so tools/ab/libq8_new.so > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lars.csv python bench.py --workload lars_resnet50 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
grep -v "^==" $O/launches_lars.csv | awk -F'","' '{print $5, $NF}' | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 4 -c 1 -o /tmp/cfg3_full python bench.py --workload cfg3_resnet50 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu3 $?
ncu -i /tmp/cfg3_full.ncu-rep --page source --csv --print-source sass > $O/cfg3_source.csv 2>/dev/null; echo src $?
python tools/ncu_stalls.py $O/cfg3_source.csv 40 > $O/cfg3_stalls.txt 2>&1; cat $O/cfg3_stalls.txt | head -70
python tools/ncu_metrics.py /tmp/cfg3_full.ncu-rep 25557032 > $O/ncu_cfg3.txt 2>&1; grep -E "gpu__time|stalls|inst_exec" $O/ncu_cfg3.txt
