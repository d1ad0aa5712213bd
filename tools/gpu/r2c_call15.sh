# Plans of <= 192 non-empty tensors launch with the 192-entry descriptor table: plan / optimizer parity, the
# full GPU suite, ABBA A/B on cfg3 (161 ResNet-50 tensors through one plan launch) and LARS.
# (result: cfg3 61.05 -> 59.52 us over six ABBA pairs, 0.77 -> 0.79; full GPU suite green; kept)
O=gpurun_out/r2c15; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "cfg3_resnet50" 30 tools/ab/libq8_small.so tools/ab/libq8_small2.so 6 > $O/ab.txt 2>&1; cat $O/ab.txt
