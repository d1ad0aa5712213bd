"""Quick device-timed probe of the fused step on a flat buffer (development tool)."""
import argparse
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2110_02861_b200 as q8
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=synth.workload_numel("cfg4_gpt2_xl"))
ap.add_argument("--kind", default="adamw")
ap.add_argument("--gdt", default="bfloat16")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
n = a.n
dev = "cuda"
p = synth.params(n, device=dev)
gs = [synth.grads(n, step=t, dtype=a.gdt, device=dev) for t in (1, 2)]
s1, a1 = synth.zero_state(n, device=dev)
s2, a2 = synth.zero_state(n, device=dev)
hp = dict(synth.HPARAMS[a.kind])
for t in range(1, 11):
    q8.optim8bit_step(a.kind, p, gs[t % 2], s1, s2, a1, a2, step=t, **hp)
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for t in range(11, 11 + a.iters):
    q8.optim8bit_step(a.kind, p, gs[t % 2], s1, s2, a1, a2, step=t, **hp)
en.record()
torch.cuda.synchronize()
ms = st.elapsed_time(en) / a.iters
gb = 2 if a.gdt != "float32" else 4
bpp = 8 + gb + (2 if a.kind == "momentum" else 4) + (16 if a.kind != "momentum" else 8) / 2048
print(json.dumps(dict(n=n, kind=a.kind, gdt=a.gdt, ms=ms, gparams_s=n / ms / 1e6, gbs=n * bpp / ms / 1e6,
                      frac=n * bpp / ms / 1e6 / 6549.1)))
