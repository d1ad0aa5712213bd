python -c "import __graft_entry__ as g; g.build()" > /dev/null
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_quantiles.py -q -k "gaussian and (17 or 4097 or 100003)" > gpurun_out/san_q.log 2>&1; echo "quantiles memcheck rc=$?"; tail -3 gpurun_out/san_q.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_quantiles.py -q -k "gaussian and (4097 or 100003)" > gpurun_out/san_qr.log 2>&1; echo "quantiles racecheck rc=$?"; tail -3 gpurun_out/san_qr.log
