set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_normalizer.py tests/test_gpu_quantiles.py -q -x -p no:cacheprovider > gpurun_out/r2/pytest_codec.log 2>&1; echo pytest $?
tail -5 gpurun_out/r2/pytest_codec.log
timeout 600 python bench.py --workload codec_gpt2_xl --steps 30 --warmup 5 > gpurun_out/r2/bench_codec2.json 2> gpurun_out/r2/bench_codec2.err; echo bench $?
tail -c 2500 gpurun_out/r2/bench_codec2.json; tail -3 gpurun_out/r2/bench_codec2.err
