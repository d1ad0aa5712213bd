"""Seeded random sweep of the fused step against the oracle (bit for bit): random sizes (incl. ragged
tails and multi-block sub-block reuse), kinds, gradient dtypes, hyper-parameters (lr, betas, eps,
weight decay, bias correction), step indices, state scales spanning many binades and gradient
scales from tiny to large -- the cases a hand-picked list misses (readings G6-G13)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

DEV = "cuda"
KINDS = ["adam", "adamw", "momentum"]
GDTS = ["float32", "float16", "bfloat16"]


@pytest.fixture(scope="module")
def q8():
    import paper_2110_02861_b200 as m
    return m


def _bits(a):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return a.view(np.uint32) if a.dtype == np.float32 else a


def _case(i):
    rng = np.random.default_rng(1000 + i)
    kind = KINDS[i % 3]
    gdt = GDTS[(i // 3) % 3]
    n = int(rng.choice([int(rng.integers(1, 4096)), int(rng.integers(4096, 200_000)),
                        2048 * int(rng.integers(600, 1500)) + int(rng.integers(0, 2048))]))
    hp = dict(lr=float(10 ** rng.uniform(-5, -0.5)), beta1=float(rng.choice([0.0, 0.5, 0.9, 0.99])),
              beta2=float(rng.choice([0.9, 0.99, 0.995, 0.999, 0.9999])), eps=float(10 ** rng.uniform(-10, -4)),
              weight_decay=float(rng.choice([0.0, 1e-4, 0.01, 0.1])), bias_correction=bool(rng.integers(0, 2)))
    step = int(rng.choice([1, 2, 7, 100, 12345]))
    gscale = float(10 ** rng.uniform(-8, 1))
    sscale = (float(10 ** rng.uniform(-12, 0)), float(10 ** rng.uniform(-20, 0)))
    return kind, gdt, n, hp, step, gscale, sscale


@pytest.mark.parametrize("i", range(90))
def test_random_case_bit_exact(q8, i):
    kind, gdt, n, hp, step, gscale, sscale = _case(i)
    p = synth.params(n, seed=i)
    s1, a1 = synth.random_state(n, seed=i + 1, scale=sscale[0])
    s2, a2 = synth.random_state(n, seed=i + 2, scale=sscale[1])
    g = synth.grads(n, step=step, seed=i, dtype="float32", std=gscale).to(synth._TORCH_DT[gdt])
    gp = [t.to(DEV).clone() for t in (p, s1, a1, s2, a2)]
    cp = [t.numpy().copy() for t in (p, s1, a1, s2, a2)]
    q8.optim8bit_step(kind, gp[0], g.to(DEV), gp[1], gp[3], gp[2], gp[4], step=step, **hp)
    oracle.optim8bit_step(kind, cp[0], synth.to_f32_numpy(g), cp[1], cp[3], cp[2], cp[4], step=step, nthreads=8, **hp)
    torch.cuda.synchronize()
    names = ["p", "s1", "absmax1"] + (["s2", "absmax2"] if kind != "momentum" else [])
    for k, name in enumerate(["p", "s1", "absmax1", "s2", "absmax2"]):
        if name not in names:
            continue
        a, b = _bits(gp[k]), _bits(cp[k])
        bad = np.nonzero(a != b)[0]
        assert bad.size == 0, f"case {i} ({kind}, {gdt}, n={n}, hp={hp}, step={step}): {name} differs at {bad[:5]}"


@pytest.mark.parametrize("i", range(12))
def test_random_tensor_list_bit_exact(q8, i):
    # one multi-tensor launch over a random list (per-tensor blocks) == per-tensor oracle steps
    rng = np.random.default_rng(5000 + i)
    kind, gdt = KINDS[i % 3], GDTS[(i // 3) % 3]
    sizes = [int(rng.integers(1, 3 * 2048)) for _ in range(int(rng.integers(2, 60)))]
    hp = dict(synth.HPARAMS[kind])
    step = int(rng.integers(1, 50))
    ents, refs = [], []
    for k, n in enumerate(sizes):
        p = synth.params(n, seed=100 * i + k)
        s1, a1 = synth.random_state(n, seed=100 * i + k + 1, scale=1e-3)
        s2, a2 = synth.random_state(n, seed=100 * i + k + 2, scale=1e-6)
        g = synth.grads(n, step=step, seed=100 * i + k, dtype=gdt)
        dev = [t.to(DEV).clone() for t in (p, g, s1, s2, a1, a2)]
        ents.append(tuple(dev[:3]) + ((dev[3],) if kind != "momentum" else (None,)) + (dev[4],)
                    + ((dev[5],) if kind != "momentum" else (None,)))
        refs.append([t.numpy().copy() for t in (p, s1, a1, s2, a2)] + [synth.to_f32_numpy(g)])
    q8.optim8bit_step_multi(kind, ents, step=step, **hp)
    torch.cuda.synchronize()
    for k, (e, r) in enumerate(zip(ents, refs)):
        oracle.optim8bit_step(kind, r[0], r[5], r[1], r[3], r[2], r[4], step=step, **hp)
        pairs = [(e[0], r[0]), (e[2], r[1]), (e[4], r[2])] + ([(e[3], r[3]), (e[5], r[4])] if kind != "momentum" else [])
        for a, b in pairs:
            assert np.array_equal(_bits(a), _bits(b)), f"list {i} tensor {k} (n={sizes[k]}, {kind}, {gdt})"
