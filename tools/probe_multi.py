"""Probe (development tool): where the multi-tensor (plan) step loses time against the flat kernel at the cfg3 size.
8-bit Momentum, fp16 grads, the bench's clean L2 flush before each timed step, time between CUDA events:
  resnet50    the 161 ResNet-50 tensors (99 below one block; every tensor has a short last block)
  rounded     161 tensors, each rounded UP to a multiple of 2048 (no short blocks; same tensor count)
  one         the same total as ONE tensor through the plan (multi-tensor kernel, one descriptor)
  flat        the flat kernel on one tensor of the same total"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_02861_b200 as q8  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
hp = dict(synth.HPARAMS["momentum"])
hpo = q8.hparams(**hp)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush2 = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)


def make(sizes):
    offs, o = [], 0
    for n in sizes:
        offs.append(o)
        o += (n + 15) // 16 * 16
    p = synth.params(o, device=dev)
    g = synth.grads(o, step=1, dtype="float16", device=dev)
    s1 = torch.zeros(o, dtype=torch.uint8, device=dev)
    a1 = torch.zeros(sum((n + 2047) // 2048 for n in sizes), dtype=torch.float32, device=dev)
    ents, bo = [], 0
    for n, off in zip(sizes, offs):
        nb = (n + 2047) // 2048
        ents.append((p[off:off + n], g[off:off + n], s1[off:off + n], None, a1[bo:bo + nb], None))
        bo += nb
    return q8.Plan("momentum", ents), (p, g, s1, a1)


def timed(fn, k=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for i in range(k):
        flush.fill_(i & 0xff)
        flush2.max()
        ev[i][0].record()
        fn()
        ev[i][1].record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3


sizes = [synth.numel(s) for s in synth.resnet50_shapes()]
total = sum(sizes)
rounded = [(n + 2047) // 2048 * 2048 for n in sizes]
t = [0]
res = {}
for name, sz in (("resnet50", sizes), ("rounded", rounded), ("one", [total])):
    plan, keep = make(sz)

    def step():
        t[0] += 1
        plan.step(hpo, t[0])
    res[name] = (round(timed(step), 1), sum(sz))
    del plan, keep
pf = synth.params(total, device=dev)
gf = synth.grads(total, step=1, dtype="float16", device=dev)
s1f = torch.zeros(total, dtype=torch.uint8, device=dev)
a1f = torch.zeros((total + 2047) // 2048, dtype=torch.float32, device=dev)


def step_flat():
    t[0] += 1
    q8.optim8bit_step("momentum", pf, gf, s1f, None, a1f, None, step=t[0], hp=hpo, lr=hp["lr"])


res["flat"] = (round(timed(step_flat), 1), total)
for k, (us, n) in res.items():
    print(f"{k:9s} {us:7.1f} us  {n:,} params  {n / us / 1e3:.3f} Gparams/ms")
