# find_tensor: next-tensor fast path before the binary search. Multi-tensor parity, probe, A/B of cfg3/LARS/LAMB.
O=gpurun_out/r2b15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py tests/test_gpu_layerwise.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log
timeout 600 python tools/probe_multi.py > $O/probe_multi.txt 2>&1; cat $O/probe_multi.txt
Q8_LIB_PATH=tools/ab/libq8_s3b.so timeout 600 python tools/probe_multi.py > $O/probe_multi_old.txt 2>&1; cat $O/probe_multi_old.txt
bash tools/ab_work.sh "cfg3_resnet50 lars_resnet50 lamb_gpt2_xl" 30 tools/ab/libq8_s3b.so tools/ab/libq8_new.so > $O/ab.txt 2>&1; cat $O/ab.txt
