"""Sustained copy bandwidth (development tool): torch b.copy_(a) over 1 Gi bf16 elements, back to back
for ~N iterations (read+write bytes), CUDA events; compare with MEASURED_PEAKS' best-of-10 burst."""
import statistics
import sys

import torch

n = 1 << 30
a = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
b = torch.empty_like(a)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 400
for _ in range(5):
    b.copy_(a)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
for i in range(iters):
    ev[i][0].record()
    b.copy_(a)
    ev[i][1].record()
torch.cuda.synchronize()
ms = [x.elapsed_time(y) for x, y in ev]
gbs = [2 * n * 2 / (m / 1e3) / 1e9 for m in ms]
print(f"copy: first {statistics.mean(gbs[:10]):.1f} GB/s, last {statistics.mean(gbs[-50:]):.1f} GB/s, "
      f"best {max(gbs):.1f}, median {statistics.median(gbs):.1f} ({iters} x {4 * n / 2**30:.0f} GiB moved)")
