"""Kernel timeline of a few steps of a bench workload under torch.profiler (CUPTI activity records: start
and end of every kernel on the device clock), printing each q8 kernel's duration and the idle gap before
it (development tool).  usage: python tools/probe_timeline.py [workload] [steps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_02861_b200 as q8  # noqa: E402
import synth  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "lamb_gpt2_xl"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = synth.WORKLOADS[wl]
kind, gdt = cfg["kind"], cfg["grad_dtype"]
hp = dict(synth.HPARAMS[kind])
eta = hp.pop("trust_coefficient", 0.001)
sizes = [synth.numel(s) for s in cfg["shapes"]]
dev = "cuda"
two = kind == "lamb"
offs, o = [], 0
for n in sizes:
    offs.append(o)
    o += (n + 15) // 16 * 16
p = synth.params(o, seed=1, device=dev)
g = synth.grads(o, step=1, dtype=gdt, device=dev)
nbt = sum((n + 2047) // 2048 for n in sizes)
s1 = torch.zeros(o, dtype=torch.uint8, device=dev)
s2 = torch.zeros(o if two else 0, dtype=torch.uint8, device=dev)
a1 = torch.zeros(nbt, dtype=torch.float32, device=dev)
a2 = torch.zeros(nbt if two else 0, dtype=torch.float32, device=dev)
ents, bo = [], 0
for n, off in zip(sizes, offs):
    nb = (n + 2047) // 2048
    ents.append((p[off:off + n], g[off:off + n], s1[off:off + n], s2[off:off + n] if two else None,
                 a1[bo:bo + nb], a2[bo:bo + nb] if two else None))
    bo += nb
tl = q8.TensorList(ents)
ws = torch.zeros(q8.layerwise_workspace_bytes(tl), dtype=torch.uint8, device=dev)
hpo = q8.hparams(**hp)
for t in range(1, 4):
    q8.optim8bit_step_layerwise(kind, tl, lr=hp["lr"], step=t, hp=hpo, trust_coefficient=eta, workspace=ws)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for t in range(4, 4 + steps):
        q8.optim8bit_step_layerwise(kind, tl, lr=hp["lr"], step=t, hp=hpo, trust_coefficient=eta, workspace=ws)
    torch.cuda.synchronize()
evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA), key=lambda e: e.time_range.start)
prev = None
tot_gap = tot_k = 0.0
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    gap = (s - prev) if prev is not None else 0.0
    print(f"{e.name[:70]:70s} dur {t - s:9.1f} us  gap {gap:7.1f} us")
    tot_k += t - s
    tot_gap += gap
    prev = t
print(f"kernels {tot_k:.1f} us, gaps {tot_gap:.1f} us over {steps} steps")
