"""Probe (development tool): pinned-host <-> device copy rates on this box -- H2D alone, D2H alone, both at once
(separate streams), 256 MB copies -- the ceiling of bench.py's host-buffer e2e path."""
import time
import torch

n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return reps * n / dt / 1e9


for _ in range(2):
    print(f"H2D alone {run(True, False):.1f} GB/s | D2H alone {run(False, True):.1f} GB/s | "
          f"both: {run(True, True):.1f} GB/s each direction")
