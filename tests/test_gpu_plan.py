"""GPU tests of prepared multi-tensor steps (q8_plan_*): 8-bit- and 32-bit-state tensors in the SAME
launch (the Stable Embedding keeps 32-bit states, S3.3 P:124-125), host-stepped and device-stepped
(capturable) plans, the device-computed scalars of G8-G10 against the host's, and a CUDA-graph
captured AdamW8bit.step() replayed against the oracle -- all bit for bit."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def q8():
    import paper_2110_02861_b200 as m
    return m


def _sizes(seed, count):
    rng = np.random.default_rng(seed)
    return [int(x) for x in rng.choice([1, 17, 64, 2047, 2048, 2049, 5000, 3 * 2048 + 5, 40_000], size=count)]


def _make(kind, gdt, sizes, bits32_every, seed):
    """Tensors alternating between 8-bit states (random codes/absmax) and 32-bit states (random fp32
    m, r >= 0); returns GPU entries (e8, e32) and the oracle's copies in plan order."""
    two = kind != "momentum"
    e8, e32, ref8, ref32 = [], [], [], []
    for i, n in enumerate(sizes):
        p = synth.params(n, seed=seed + i)
        if i % bits32_every == bits32_every - 1:
            m = synth.params(n, seed=seed + 500 + i, std=1e-3)
            r = synth.params(n, seed=seed + 900 + i, std=1e-6).abs()
            e32.append([p.to(DEV), None, m.to(DEV), r.to(DEV) if two else None])
            ref32.append([p.numpy().copy(), m.numpy().copy(), r.numpy().copy()])
        else:
            s1, a1 = synth.random_state(n, seed=seed + 100 + i, scale=1e-3)
            s2, a2 = synth.random_state(n, seed=seed + 200 + i, scale=1e-6)
            e8.append([p.to(DEV), None, s1.to(DEV), s2.to(DEV) if two else None, a1.to(DEV), a2.to(DEV) if two else None])
            ref8.append([p.numpy().copy(), s1.numpy().copy(), s2.numpy().copy(), a1.numpy().copy(), a2.numpy().copy()])
    return e8, e32, ref8, ref32


def _oracle_step(kind, ref8, ref32, g8, g32, t, hp):
    two = kind != "momentum"
    for r, g in zip(ref8, g8):
        oracle.optim8bit_step(kind, r[0], g, r[1], r[2] if two else None, r[3], r[4] if two else None, step=t, **hp)
    for r, g in zip(ref32, g32):
        oracle.optim32bit_step(kind, r[0], g, r[1], r[2] if two else None, step=t, **hp)


def _assert_same(kind, e8, e32, ref8, ref32):
    two = kind != "momentum"
    for i, (e, r) in enumerate(zip(e8, ref8)):
        assert np.array_equal(e[0].cpu().numpy().view(np.uint32), r[0].view(np.uint32)), f"8-bit p {i}"
        assert np.array_equal(e[2].cpu().numpy(), r[1]), f"s1 {i}"
        assert np.array_equal(e[4].cpu().numpy().view(np.uint32), r[3].view(np.uint32)), f"absmax1 {i}"
        if two:
            assert np.array_equal(e[3].cpu().numpy(), r[2]), f"s2 {i}"
            assert np.array_equal(e[5].cpu().numpy().view(np.uint32), r[4].view(np.uint32)), f"absmax2 {i}"
    for i, (e, r) in enumerate(zip(e32, ref32)):
        assert np.array_equal(e[0].cpu().numpy().view(np.uint32), r[0].view(np.uint32)), f"32-bit p {i}"
        assert np.array_equal(e[2].cpu().numpy().view(np.uint32), r[1].view(np.uint32)), f"m {i}"
        if two:
            assert np.array_equal(e[3].cpu().numpy().view(np.uint32), r[2].view(np.uint32)), f"r {i}"


@pytest.mark.parametrize("count", [450, 192])
@pytest.mark.parametrize("kind,gdt,device_step", [("adamw", "bfloat16", False), ("adam", "float16", True),
                                                  ("momentum", "float32", False), ("adamw", "float32", True),
                                                  ("momentum", "bfloat16", True)])
def test_mixed_plan_matches_oracle(q8, kind, gdt, device_step, count):
    """450 tensors (two launches of <= 384) or 192 (one launch with the 192-entry descriptor table,
    q8_launch.h kSmallMaxT), every third one with 32-bit states, 3 steps."""
    hp = dict(synth.HPARAMS[kind])
    if kind == "adam":
        hp["weight_decay"] = 1e-3      # L2 variant of the kernel
    sizes = _sizes(11, count)
    e8, e32, ref8, ref32 = _make(kind, gdt, sizes, 3, seed=3)
    step_t = torch.zeros(1, dtype=torch.int64, device=DEV)
    plan = None
    hpo = q8.hparams(**hp)
    for t in range(1, 4):
        g8 = [synth.grads(e[0].numel(), step=t, seed=i, dtype=gdt) for i, e in enumerate(e8)]
        g32 = [synth.grads(e[0].numel(), step=t, seed=1000 + i, dtype=gdt) for i, e in enumerate(e32)]
        for e, g in zip(e8, g8):
            e[1] = g.to(DEV)
        for e, g in zip(e32, g32):
            e[1] = g.to(DEV)
        if plan is None:
            plan = q8.Plan(kind, [tuple(e) for e in e8], [tuple(e) for e in e32])
        plan.set_grads([e[1] for e in e8] + [e[1] for e in e32])
        if device_step:
            plan.step_device(hpo, step_t)
        else:
            plan.step(hpo, t)
        torch.cuda.synchronize()
        _oracle_step(kind, ref8, ref32, [synth.to_f32_numpy(g) for g in g8], [synth.to_f32_numpy(g) for g in g32], t,
                     hp)
        _assert_same(kind, e8, e32, ref8, ref32)
    if device_step:
        assert int(step_t.item()) == 3


@pytest.mark.parametrize("kind,hpkey", [("adam", "adam"), ("adamw", "adamw"), ("adam", "adam_paper"),
                                        ("lamb", "lamb"), ("momentum", "momentum")])
def test_device_scalars_equal_host(q8, kind, hpkey):
    """compute_scalars on the device (the capturable path) == on the host, for every step 1..2^16
    and 2^14 sampled steps up to 2^40 (pow() implementations differ; the fp32 results may not)."""
    hp = dict(synth.HPARAMS[hpkey])
    hp.pop("trust_coefficient", None)
    hpo = q8.hparams(**hp)
    rng = np.random.default_rng(5)
    steps = np.concatenate([np.arange(1, 1 << 16), rng.integers(1 << 16, 1 << 40, 1 << 14)]).astype(np.int64)
    dev = q8.step_scalars_device(kind, hpo, torch.from_numpy(steps).to(DEV)).cpu().numpy()
    host = np.stack([q8.step_scalars(kind, hpo, int(t)).numpy() for t in steps])
    bad = np.nonzero(np.any(dev.view(np.uint32) != host.view(np.uint32), axis=1))[0]
    assert bad.size == 0, (steps[bad[:5]], dev[bad[:2]], host[bad[:2]])


def test_cuda_graph_replay_matches_oracle(q8):
    """AdamW8bit(capturable=True) over a model with a StableEmbedding (32-bit states) and Linear layers
    (8-bit states): step() captured once in a CUDA graph, replayed with new gradients copied into the
    captured gradient buffers; every replay equals the oracle bit for bit and advances the device
    step counter (no host work per replay)."""
    torch.manual_seed(0)
    emb = q8.StableEmbedding(500, 64).to(DEV)
    lin = torch.nn.Linear(64, 3000).to(DEV)
    params = list(emb.parameters()) + list(lin.parameters())
    hp = dict(lr=2e-3, beta1=0.9, beta2=0.99, eps=1e-7, weight_decay=0.01, bias_correction=True)
    opt = q8.AdamW8bit(params, lr=hp["lr"], betas=(hp["beta1"], hp["beta2"]), eps=hp["eps"],
                       weight_decay=hp["weight_decay"], capturable=True)
    for i, p in enumerate(params):
        p.grad = synth.grads(p.numel(), step=0, seed=i).to(DEV).view_as(p)
    bits = [32 if getattr(p, "_q8_optim_bits", 8) == 32 else 8 for p in params]
    ref = [p.detach().cpu().numpy().reshape(-1).copy() for p in params]
    st = [dict(s1=np.zeros(r.size, np.uint8), s2=np.zeros(r.size, np.uint8),
               a1=np.zeros((r.size + 2047) // 2048, np.float32), a2=np.zeros((r.size + 2047) // 2048, np.float32),
               m=np.zeros(r.size, np.float32), r=np.zeros(r.size, np.float32)) for r in ref]

    def oracle_step(t, grads):
        for r, g, s, b in zip(ref, grads, st, bits):
            if b == 32:
                oracle.optim32bit_step("adamw", r, g, s["m"], s["r"], step=t, **hp)
            else:
                oracle.optim8bit_step("adamw", r, g, s["s1"], s["s2"], s["a1"], s["a2"], step=t, **hp)

    def check():
        for p, r in zip(params, ref):
            assert np.array_equal(p.detach().cpu().numpy().reshape(-1).view(np.uint32), r.view(np.uint32))

    # warm-up eager step on a side stream (builds the plan and the state), as torch.cuda.graph requires
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        opt.step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    oracle_step(1, [p.grad.cpu().numpy().reshape(-1) for p in params])
    check()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        opt.step()
    for t in range(2, 7):
        new = [synth.grads(p.numel(), step=t, seed=i) for i, p in enumerate(params)]
        for p, x in zip(params, new):
            p.grad.copy_(x.to(DEV).view_as(p))
        g.replay()
        torch.cuda.synchronize()
        oracle_step(t, [x.numpy() for x in new])
        check()
    assert int(opt.state[params[0]]["step"].item()) == 6


def test_optimizer_state_reset_rebuilds_plan(q8):
    """a state that is cleared or replaced must not keep being stepped through a cached
    plan: after opt.state.clear() the next step starts from zero state at step 1 (== a fresh
    optimizer), bit for bit."""
    torch.manual_seed(1)
    lin = torch.nn.Linear(100, 3000).to(DEV)
    lin2 = torch.nn.Linear(100, 3000).to(DEV)
    lin2.load_state_dict(lin.state_dict())
    o1 = q8.AdamW8bit(lin.parameters(), lr=1e-3)
    x = torch.randn(16, 100, device=DEV)
    for _ in range(2):
        o1.zero_grad()
        lin(x).square().mean().backward()
        o1.step()
    o1.state.clear()
    lin2.load_state_dict(lin.state_dict())
    o2 = q8.AdamW8bit(lin2.parameters(), lr=1e-3)
    for m, o in ((lin, o1), (lin2, o2)):
        o.zero_grad()
        m(x).square().mean().backward()
        o.step()
    for a, b in zip(lin.parameters(), lin2.parameters()):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    assert o1.state_dict()["state"][0]["step"] == 1
