# Layer-wise lists of <= 192 tensors launch with a 192-entry descriptor table (13.8 KB of kernel parameters
# instead of 26 KB): layer-wise + optimizer-API parity, ABBA A/B on LARS over ResNet-50 (161 tensors, two launches).
# (result: 89.63 -> 88.29 us over six ABBA pairs, LARS 0.784 -> 0.796; kept)
O=gpurun_out/r2c14; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layerwise.py tests/test_gpu_optim.py tests/test_abi.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "lars_resnet50" 30 tools/ab/libq8_new2.so tools/ab/libq8_small.so 6 > $O/ab.txt 2>&1; cat $O/ab.txt
