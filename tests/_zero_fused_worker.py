"""Worker of tests/test_gpu_zero_fused.py: one rank of the fused ZeRO-1 step.  Launched by
torchrun with every rank on cuda:0 (processes share one GPU, gloo for the host exchange); each
rank writes its full parameter buffer and its shard states after every step to OUT_DIR."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_02861_b200 as q8  # noqa: E402
import synth  # noqa: E402


def main():
    out_dir, n, kind, gdt, steps, ctas = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5]), \
        int(sys.argv[6])
    mode = sys.argv[7] if len(sys.argv) > 7 else "shared"
    if mode == "nvls":   # one GPU per rank, NCCL, symmetric memory with NVLS multicast (required)
        local = int(os.environ["LOCAL_RANK"])
        dev = torch.device("cuda", local)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=dev)
    else:                # every rank on cuda:0, gloo for the host exchange, CUDA IPC peer mappings
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo")
    rank = dist.get_rank()
    hp = dict(synth.HPARAMS[kind])
    zo = q8.ZeroFusedOptimizer8bit(n, kind=kind, grad_dtype=getattr(torch, gdt), device=dev, num_ctas=ctas,
                                   multicast="on" if mode == "nvls" else "off", **hp)
    assert (zo.p_mc is not None) == (mode == "nvls")
    zo.params[:n] = synth.params(n, seed=3).to(dev)
    torch.cuda.synchronize()
    dist.barrier()
    for t in range(1, steps + 1):
        zo.grads.zero_()
        zo.grads[:n] = synth.grads(n, step=t, seed=50 + rank, dtype=gdt).to(dev)
        torch.cuda.synchronize()
        dist.barrier()          # (a real trainer needs no host barrier: the kernel's flags order the ranks)
        zo.step()
        torch.cuda.synchronize()
        np.savez(os.path.join(out_dir, f"r{rank}_t{t}.npz"), p=zo.params.cpu().numpy(), s1=zo.s1.cpu().numpy(),
                 a1=zo.absmax1.cpu().numpy(),
                 s2=zo.s2.cpu().numpy() if zo.s2 is not None else np.zeros(0, np.uint8),
                 a2=zo.absmax2.cpu().numpy() if zo.absmax2 is not None else np.zeros(0, np.float32))
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
