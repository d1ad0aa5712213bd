set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 120 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/probe_nccl_shared.py > gpurun_out/r2/nccl_probe.log 2>&1; echo probe $?
tail -20 gpurun_out/r2/nccl_probe.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-e2e > gpurun_out/r2/bench_base.json 2> gpurun_out/r2/bench_base.err; echo bench $?
cat gpurun_out/r2/bench_base.json
