# Staged short last blocks + find_tensor next-tensor fast path, together: multi-tensor parity, ABBA A/B.
O=gpurun_out/r2b19; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py tests/test_gpu_layerwise.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "cfg3_resnet50" 50 tools/ab/libq8_s3c.so tools/ab/libq8_new.so 8 > $O/ab_cfg3.txt 2>&1; cat $O/ab_cfg3.txt
bash tools/ab_work.sh "lars_resnet50 lamb_gpt2_xl" 20 tools/ab/libq8_s3c.so tools/ab/libq8_new.so 4 > $O/ab_lw.txt 2>&1; cat $O/ab_lw.txt
