set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_zero_fused.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "zero_fused or multirank or tensorwise or exhaustive or quantize or codec or linear" > gpurun_out/r2/pytest_zero.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2/pytest_zero.log
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-zero1 --zero-fused --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2/bench_zero_w1.json 2> gpurun_out/r2/bench_zero_w1.err; echo zero $?
tail -c 1500 gpurun_out/r2/bench_zero_w1.json
timeout 600 python bench.py --workload codec_gpt2_xl --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench_codec3.json 2> gpurun_out/r2/bench_codec3.err; echo codec $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 4 -c 1 -o gpurun_out/r2/cfg3_full python bench.py --workload cfg3_resnet50 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_cfg3.log 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim8bit_step -s 4 -c 1 -o gpurun_out/r2/cfg2_full python bench.py --workload cfg2_gpt2_medium --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2/ncu_cfg2.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quantize_tma -s 2 -c 1 -o gpurun_out/r2/codec_full python bench.py --workload codec_gpt2_xl --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2/ncu_codec.log 2>&1; echo ncuc $?
