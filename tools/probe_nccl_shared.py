"""Probe: can NCCL form a process group when several ranks share one GPU (world > device count)?
Run under torchrun on a one-GPU box; prints one line per rank."""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
try:
    dist.init_process_group("nccl", device_id=dev)
    x = torch.full((1024,), float(rank + 1), device=dev)
    dist.all_reduce(x)
    y = torch.empty(1024 * dist.get_world_size(), device=dev)
    dist.all_gather_into_tensor(y, x)
    torch.cuda.synchronize()
    print(f"rank {rank}: nccl shared-GPU ok, allreduce={float(x[0])}", flush=True)
    dist.destroy_process_group()
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: nccl shared-GPU FAILED: {type(e).__name__}: {str(e)[:300]}", flush=True)
