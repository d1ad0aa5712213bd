# compute-sanitizer memcheck over the whole GPU suite except the long sweeps (final round-2 state).
O=gpurun_out/r2mc; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 3000 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider \
  -k "not all_mantissas and not binades and not fullsize and not exhaustive and not multirank" > $O/memcheck_all.log 2>&1
echo "memcheck rc=$?: $(grep -E 'passed|failed' $O/memcheck_all.log | tail -1) | $(grep -E 'ERROR SUMMARY' $O/memcheck_all.log | tail -1)"
