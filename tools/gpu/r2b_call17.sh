# New layer-wise workspace test + the full layer-wise file.
O=gpurun_out/r2b17; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_layerwise.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest $?
tail -3 $O/pytest.log; grep -E "^E " $O/pytest.log | head
