# Round 2 sanitizer pass (run on a gpurun box): memcheck on the kernels added or changed this round,
# racecheck on the TMA stage-reuse reproducer (tools/micro/racecheck_tma_repro.cu) in both hand-off modes.
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/rc_repro tools/micro/racecheck_tma_repro.cu
for m in 0 1; do
  timeout 300 compute-sanitizer --tool racecheck --print-limit 4 /tmp/rc_repro $m > gpurun_out/r2/san_repro_mode$m.log 2>&1
  echo "racecheck repro mode $m rc=$?: $(grep -E '^mode' gpurun_out/r2/san_repro_mode$m.log) | $(grep -E 'RACECHECK SUMMARY' gpurun_out/r2/san_repro_mode$m.log | tail -1)"
done
run() { tool=$1; shift; name=$1; shift; timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -p no:cacheprovider "$@" > gpurun_out/r2/san_${tool}_${name}.log 2>&1; echo "$tool $name rc=$?: $(grep -E 'passed|failed' gpurun_out/r2/san_${tool}_${name}.log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r2/san_${tool}_${name}.log | tail -1)"; }
run memcheck plan tests/test_gpu_plan.py -k "mixed or graph or reset"
run memcheck layerwise tests/test_gpu_layerwise.py
run memcheck codec tests/test_gpu_parity.py -k "quantize or tensorwise or linear or dequantize"
run memcheck zero tests/test_gpu_zero_fused.py -k "single_rank"
run memcheck normalizer tests/test_gpu_normalizer.py -k "vs_oracle"
run synccheck layerwise tests/test_gpu_layerwise.py -k "lars"
run racecheck codec tests/test_gpu_parity.py -k "(quantize and (17 or 2049)) or linear"
