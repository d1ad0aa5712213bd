# LARS: norms pass loads p and g with L2::evict_last, the step demotes each line after staging it
# (applypriority): layer-wise parity, ABBA A/B vs HEAD (libq8_new2), CUPTI timeline.
# (result: no gain -- 90.9 vs 89.1 us over six ABBA pairs; the step kernel durations unchanged -- dropped, DESIGN 6.10)
O=gpurun_out/r2c9; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layerwise.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "lars_resnet50" 30 tools/ab/libq8_new2.so tools/ab/libq8_keep.so 6 > $O/ab.txt 2>&1; cat $O/ab.txt
Q8_LIB_PATH=tools/ab/libq8_new2.so python tools/probe_timeline.py lars_resnet50 4 > $O/tl_base.txt 2>&1
Q8_LIB_PATH=tools/ab/libq8_keep.so python tools/probe_timeline.py lars_resnet50 4 > $O/tl_keep.txt 2>&1
tail -9 $O/tl_base.txt; tail -9 $O/tl_keep.txt
