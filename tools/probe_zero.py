"""Probe (development tool): the fused ZeRO-1 kernel at world size 1 against the plain fused step on the
same cfg4-sized buffer, device-timed back to back; `--ncu` runs one launch of each (for an ncu capture)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_02861_b200 as q8  # noqa: E402
import synth  # noqa: E402

n = synth.workload_numel("cfg4_gpt2_xl")
hp = dict(synth.HPARAMS["adamw"])
iters = 1 if "--ncu" in sys.argv else 30
zf = q8.ZeroFusedOptimizer8bit(n, kind="adamw", grad_dtype=torch.bfloat16, device="cuda", multicast="off", **hp)
zf.params[:n].normal_(0, 0.02)
zf.grads[:n].normal_(0, 1e-3)
p = zf.params.clone()
g = zf.grads.clone()
s1, a1 = synth.zero_state(zf.n_pad, device="cuda")
s2, a2 = synth.zero_state(zf.n_pad, device="cuda")


def fused():
    zf.step()


t = [0]


def plain():
    t[0] += 1
    q8.optim8bit_step("adamw", p, g, s1, s2, a1, a2, step=t[0], **hp)


for f in (fused, plain):
    for _ in range(3 if iters > 1 else 1):
        f()
torch.cuda.synchronize()
res = {}
for name, f in (("fused", fused), ("plain", plain), ("fused2", fused), ("plain2", plain)):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in ev:
        a.record()
        f()
        b.record()
    torch.cuda.synchronize()
    res[name] = statistics.mean(a.elapsed_time(b) for a, b in ev)
print({k: round(v, 4) for k, v in res.items()})
