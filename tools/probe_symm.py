"""Probe torch symmetric memory on this box (development tool): world size from torchrun;
every rank uses cuda:0 when Q8_SAME_GPU=1 (two processes sharing one GPU)."""
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as sm

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
same = os.environ.get("Q8_SAME_GPU") == "1"
dev = torch.device("cuda", 0 if same else int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
backend = os.environ.get("Q8_PG", "gloo" if same else "nccl")
dist.init_process_group(backend)
try:
    print(rank, "backend", sm.get_backend(dev), flush=True)
except Exception as e:
    print(rank, "get_backend err", e, flush=True)
try:
    t = sm.empty(1 << 20, dtype=torch.float32, device=dev)
    h = sm.rendezvous(t, dist.group.WORLD)
    try:
        mc = sm._SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, dev.index)
    except Exception as e:
        mc = repr(e)
    print(rank, "rendezvous ok", "mc", mc, "mcptr", getattr(h, "multicast_ptr", None), "ptrs", list(h.buffer_ptrs), "sig", list(h.signal_pad_ptrs),
          "sigsize", h.signal_pad_size, flush=True)
    t.fill_(rank + 1)
    torch.cuda.synchronize()
    dist.barrier()
    peer = h.get_buffer((rank + 1) % world, (4,), torch.float32)
    print(rank, "peer values", peer.tolist(), flush=True)
except Exception as e:
    import traceback
    traceback.print_exc()
dist.barrier()
dist.destroy_process_group()
