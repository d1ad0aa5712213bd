# LARS norms+scale fused (two launches, PDL step) + staged tails: layer-wise parity, then A/B vs HEAD.
O=gpurun_out/r2b4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo pytest $?
tail -3 $O/pytest.log
bash tools/ab_work.sh "cfg3_resnet50 lars_resnet50 lamb_gpt2_xl" 30 tools/ab/libq8_head.so tools/ab/libq8_new.so > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lars.csv python bench.py --workload lars_resnet50 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
grep -v "^==" $O/launches_lars.csv | awk -F'","' '{print $5, $NF}' | tail -6
