python -c "import __graft_entry__ as g; g.build()" > /dev/null
Q8_OBJDIR=/tmp/q8_probe Q8_EXTRA_NVCC_FLAGS="-DQ8_NORMS_BARRIER_PROBE" Q8_LIB_OUT=/tmp/libq8_probe.so python paper_2110_02861_b200/build.py --force > /dev/null
Q8_LIB_PATH=/tmp/libq8_probe.so timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -q -p no:cacheprovider tests/test_gpu_layerwise.py > gpurun_out/san4_probe.log 2>&1; echo "probe rc=$?: $(grep -E 'passed|failed' gpurun_out/san4_probe.log | tail -1) | $(grep -E 'RACECHECK SUMMARY' gpurun_out/san4_probe.log | tail -1)"
