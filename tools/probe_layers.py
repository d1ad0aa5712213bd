"""Device-timed probe of the multi-tensor and layer-wise steps over a real layer list
(development tool): GPT-2-XL's 580 tensors as views of one flat allocation."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_02861_b200 as q8
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="lamb_gpt2_xl")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--modes", default="adamw_flat,adamw_list,lamb_list")
a = ap.parse_args()
dev = "cuda"
sizes = [synth.numel(s) for s in synth.WORKLOADS[a.workload]["shapes"]]
offs, o = [], 0
for n in sizes:
    offs.append(o)
    o += (n + 15) // 16 * 16
total = o
p = synth.params(total, device=dev)
g = synth.grads(total, step=1, dtype="bfloat16", device=dev)
s1 = torch.zeros(total, dtype=torch.uint8, device=dev)
s2 = torch.zeros(total, dtype=torch.uint8, device=dev)
nbt = sum((n + 2047) // 2048 for n in sizes)
a1 = torch.zeros(max(nbt, (total + 2047) // 2048), device=dev)
a2 = torch.zeros_like(a1)
ents, bo = [], 0
for n, off in zip(sizes, offs):
    nb = (n + 2047) // 2048
    ents.append((p[off:off + n], g[off:off + n], s1[off:off + n], s2[off:off + n], a1[bo:bo + nb], a2[bo:bo + nb]))
    bo += nb
tl = q8.TensorList(ents)
ws = torch.empty(q8.layerwise_workspace_bytes(tl), dtype=torch.uint8, device=dev)
hpw = dict(synth.HPARAMS["adamw"])
hpl = dict(synth.HPARAMS["lamb"])


def run(mode, t):
    if mode == "adamw_flat":
        q8.optim8bit_step("adamw", p, g, s1, s2, a1, a2, step=t, **hpw)
    elif mode == "adamw_list":
        q8.optim8bit_step_multi("adamw", tl, step=t, **hpw)
    elif mode == "lamb_list":
        q8.optim8bit_step_layerwise("lamb", tl, step=t, workspace=ws, **hpl)


out = {}
for mode in a.modes.split(","):
    for t in range(1, 6):
        run(mode, t)
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for t in range(6, 6 + a.iters):
        run(mode, t)
    en.record()
    torch.cuda.synchronize()
    out[mode] = st.elapsed_time(en) / a.iters
print(json.dumps(dict(n=sum(sizes), tensors=len(sizes), ms=out)))
