# LAMB norms pass with per-segment norm accumulation (one warp reduction per tensor segment): layer-wise parity, ABBA A/B vs the base build.
O=gpurun_out/r2c2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layerwise.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
bash tools/ab_work.sh "lamb_gpt2_xl" 20 tools/ab/libq8_base.so tools/ab/libq8_new.so 4 > $O/ab.txt 2>&1; cat $O/ab.txt
