set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py tests/test_gpu_layerwise.py tests/test_gpu_zero_fused.py tests/test_gpu_fuzz.py tests/test_gpu_optim.py tests/test_gpu_normalizer.py -q -x -p no:cacheprovider > gpurun_out/r2/pytest_c7.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2/pytest_c7.log
for w in cfg3_resnet50 codec_gpt2_xl lars_resnet50 lamb_gpt2_xl; do
timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench7_$w.json 2> gpurun_out/r2/bench7_$w.err; echo $w $?
done
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-zero1 --zero-fused --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2/bench7_zero_w1.json 2> gpurun_out/r2/bench7_zero_w1.err; echo zero $?
