python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() { tool=$1; shift; name=$1; shift; timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -p no:cacheprovider "$@" > gpurun_out/san2_${tool}_${name}.log 2>&1; echo "$tool $name rc=$?: $(grep -E 'passed|failed' gpurun_out/san2_${tool}_${name}.log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san2_${tool}_${name}.log | tail -1)"; }
run memcheck step tests/test_gpu_parity.py -k "test_step_single_bit_exact and (17 or 6149)"
run racecheck step tests/test_gpu_parity.py -k "test_step_single_bit_exact and 6149"
run memcheck multi tests/test_gpu_parity.py -k "multi_tensor"
run racecheck multi tests/test_gpu_parity.py -k "multi_tensor_many"
run memcheck codec tests/test_gpu_parity.py -k "(test_quantize_dequantize_bit_exact and (2049 or 17)) or (tensorwise and (17 or 2049))"
run memcheck layerwise tests/test_gpu_layerwise.py -k "matches_oracle or zero_tensors"
run racecheck layerwise tests/test_gpu_layerwise.py -k "matches_oracle"
run memcheck optim32 tests/test_gpu_optim.py -k "32bit or stable"
run memcheck zero1 tests/test_gpu_zero_fused.py -k "single_rank"
