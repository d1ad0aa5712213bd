python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() { tool=$1; shift; name=$1; shift; timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -p no:cacheprovider "$@" > gpurun_out/san3_${tool}_${name}.log 2>&1; echo "$tool $name rc=$?: $(grep -E 'passed|failed' gpurun_out/san3_${tool}_${name}.log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san3_${tool}_${name}.log | tail -1)"; }
run racecheck layerwise tests/test_gpu_layerwise.py
run racecheck optim tests/test_gpu_optim.py -k "32bit or stable or matches_oracle"
run racecheck zero1 tests/test_gpu_zero_fused.py -k "single_rank"
run racecheck codec tests/test_gpu_parity.py -k "(test_quantize_dequantize_bit_exact and (2049 or 17)) or (tensorwise and (17 or 2049)) or unsigned_negative"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
