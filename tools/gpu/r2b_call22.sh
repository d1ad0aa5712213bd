# LAMB norms pass with 3 sub-blocks x 3 TMA stages (16-bit grads): layer-wise parity, ABBA A/B, launch list.
O=gpurun_out/r2b22; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "lamb_gpt2_xl" 20 tools/ab/libq8_s3d.so tools/ab/libq8_new.so 4 > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lamb.csv python bench.py --workload lamb_gpt2_xl --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncul $?
grep -v "^==" $O/launches_lamb.csv | awk -F'","' '{print $5, $NF}' | grep q8 | tail -6
