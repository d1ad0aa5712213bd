set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_zero_fused.py tests/test_gpu_normalizer.py tests/test_gpu_layerwise.py tests/test_gpu_parity.py -x -q -k "multirank or zero_fused or normalizer or layerwise or linear or tensorwise" > gpurun_out/r2/pytest_new.log 2>&1; echo pytest $?
tail -30 gpurun_out/r2/pytest_new.log
