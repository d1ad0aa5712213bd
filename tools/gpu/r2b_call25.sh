# Multi-tensor range end in shared memory: multi/plan parity, ABBA A/B of the plan paths.
O=gpurun_out/r2b25; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py tests/test_gpu_layerwise.py tests/test_gpu_optim.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "optim_api_gpt2_xl" 40 tools/ab/libq8_s3e.so tools/ab/libq8_new.so 4 > $O/ab_api.txt 2>&1; cat $O/ab_api.txt
bash tools/ab_work.sh "cfg3_resnet50 lamb_gpt2_xl" 30 tools/ab/libq8_s3e.so tools/ab/libq8_new.so 4 > $O/ab_other.txt 2>&1; cat $O/ab_other.txt
