# Block absmax staged by the block's TMA (16-B chunk of absmax1/absmax2 into a per-stage slot) instead of a
# global load at the top of each block: full GPU suite, ABBA A/B vs HEAD (libq8_new2) on cfg4, cfg3, LAMB.
# (result: parity green, but cfg4 3.747 -> 3.885 ms and LAMB 6.95 -> 7.37 ms over four ABBA pairs, cfg3 unchanged: dropped)
O=gpurun_out/r2c13; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -5
bash tools/ab_work.sh "cfg4_gpt2_xl cfg3_resnet50 lamb_gpt2_xl" 20 tools/ab/libq8_new2.so tools/ab/libq8_abs.so 4 > $O/ab.txt 2>&1; cat $O/ab.txt
