# Sanitizer pass on the kernels changed in round 2 session 3: the LARS norms pass with per-tensor counters
# (memcheck, racecheck, synccheck), the PDL step launch, the caller-table quantizer's bucket-table build.
O=gpurun_out/r2san; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() { tool=$1; shift; name=$1; shift; timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -p no:cacheprovider "$@" > $O/san_${tool}_${name}.log 2>&1; echo "$tool $name rc=$?: $(grep -E 'passed|failed' $O/san_${tool}_${name}.log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/san_${tool}_${name}.log | tail -1)"; }
run memcheck lars tests/test_gpu_layerwise.py -k "lars or chunk or empty or zero"
run racecheck lars tests/test_gpu_layerwise.py -k "lars and not sweep and not one_launch"
run synccheck lars tests/test_gpu_layerwise.py -k "lars and not sweep"
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 20 python tools/rc_codec.py > $O/san_${tool}_codec_generic.log 2>&1
  echo "$tool codec_generic rc=$?: $(grep -E '^ok' $O/san_${tool}_codec_generic.log) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/san_${tool}_codec_generic.log | tail -1)"
done
run memcheck staged_tails tests/test_gpu_parity.py -k "staged_tails"
