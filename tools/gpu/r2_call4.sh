set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_plan.py tests/test_gpu_normalizer.py tests/test_gpu_optim.py -v --durations=10 -p no:cacheprovider > gpurun_out/r2/pytest_plan.log 2>&1; echo pytest $?
grep -E "PASS|FAIL|ERROR|passed|failed" gpurun_out/r2/pytest_plan.log | tail -40
for w in cfg4_gpt2_xl cfg3_resnet50 optim_api_gpt2_xl codec_gpt2_xl; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e > gpurun_out/r2/bench_$w.json 2> gpurun_out/r2/bench_$w.err; echo bench $w $?
  tail -c 3000 gpurun_out/r2/bench_$w.json; tail -3 gpurun_out/r2/bench_$w.err
done
timeout 600 python bench.py --workload cfg2_gpt2_medium --steps 100 --warmup 10 --no-e2e > gpurun_out/r2/bench_cfg2.json 2> gpurun_out/r2/bench_cfg2.err; echo bench cfg2 $?
tail -c 3000 gpurun_out/r2/bench_cfg2.json; tail -3 gpurun_out/r2/bench_cfg2.err
