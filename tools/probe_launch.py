"""Probe (development tool): where the cfg3 bench's event time goes beyond the kernel's own duration.
Times one multi-tensor (ResNet-50, 161 tensors) 8-bit Momentum step four ways: events right around the
plan step after an L2 flush (the bench), the same with a GPU sleep before the first event (no host
gap possible), back-to-back steps without flushes, and the flat kernel on one equally large tensor."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_02861_b200 as q8  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
shapes = synth.resnet50_shapes()
sizes = [synth.numel(s) for s in shapes]
offs, o = [], 0
for n in sizes:
    offs.append(o)
    o += (n + 15) // 16 * 16
total = o
p = synth.params(total, device=dev)
g = synth.grads(total, step=1, dtype="float16", device=dev)
s1 = torch.zeros(total, dtype=torch.uint8, device=dev)
nbt = sum((n + 2047) // 2048 for n in sizes)
a1 = torch.zeros(nbt, dtype=torch.float32, device=dev)
ents, bo = [], 0
for n, off in zip(sizes, offs):
    nb = (n + 2047) // 2048
    ents.append((p[off:off + n], g[off:off + n], s1[off:off + n], None, a1[bo:bo + nb], None))
    bo += nb
hp = dict(synth.HPARAMS["momentum"])
hpo = q8.hparams(**hp)
plan = q8.Plan("momentum", ents)
tl = q8.TensorList(ents, "momentum")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush2 = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
t = [0]


def step_plan():
    t[0] += 1
    plan.step(hpo, t[0])


def step_multi():
    t[0] += 1
    q8.optim8bit_step_multi("momentum", tl, lr=hp["lr"], step=t[0], hp=hpo)


def timed(fn, mode, k=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for i in range(k):
        if mode != "nofl":
            flush.fill_(i & 0xff)
        if mode == "clean":  # then read another 256 MB: the flush's dirty lines are written back before ev0
            flush2.max()
        if mode == "sleep":
            torch.cuda._sleep(200000)
        ev[i][0].record()
        fn()
        ev[i][1].record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3


pf = synth.params(total, device=dev)
s1f = torch.zeros(total, dtype=torch.uint8, device=dev)
a1f = torch.zeros((total + 2047) // 2048, dtype=torch.float32, device=dev)


def step_flat():
    t[0] += 1
    q8.optim8bit_step("momentum", pf, g, s1f, None, a1f, None, step=t[0], hp=hpo, lr=hp["lr"])


for name, fn in (("plan", step_plan), ("multi", step_multi), ("flat", step_flat)):
    print(name, {m: round(timed(fn, m), 1) for m in ("bench", "sleep", "nofl", "clean")}, "us")
