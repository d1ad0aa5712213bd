"""GPU tests of the torch-facing API (the paper's "two-line change", P:7): Adam8bit / AdamW8bit /
Momentum8bit over real nn.Module parameters equal per-tensor oracle steps bit for bit; state_dict
save/load resumes bit-identically; ZeRO-1 with one rank equals the plain step."""
import copy

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


def make_model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(300, 700), torch.nn.LayerNorm(700), torch.nn.Linear(700, 50)).to(DEV)


@pytest.mark.parametrize("cls,kind,extra", [("Adam8bit", "adam", {}), ("AdamW8bit", "adamw", {}),
                                            ("Momentum8bit", "momentum", {})])
def test_optimizer_matches_oracle(q8, cls, kind, extra):
    model = make_model()
    ref = [p.detach().cpu().numpy().copy() for p in model.parameters()]
    if kind == "momentum":
        opt = q8.Momentum8bit(model.parameters(), lr=0.05, momentum=0.9, weight_decay=1e-4)
        hp = dict(lr=0.05, beta1=0.9, beta2=0.0, eps=1e-8, weight_decay=1e-4, bias_correction=False)
    else:
        opt = getattr(q8, cls)(model.parameters(), lr=1e-3, betas=(0.9, 0.995), eps=1e-7, weight_decay=0.01)
        hp = dict(lr=1e-3, beta1=0.9, beta2=0.995, eps=1e-7, weight_decay=0.01, bias_correction=True)
    st = [dict(s1=np.zeros(p.size, np.uint8), s2=np.zeros(p.size, np.uint8),
               a1=np.zeros((p.size + 2047) // 2048, np.float32), a2=np.zeros((p.size + 2047) // 2048, np.float32))
          for p in ref]
    x = torch.randn(64, 300, device=DEV)
    for t in range(1, 4):
        opt.zero_grad()
        model(x).square().mean().backward()
        grads = [p.grad.detach().cpu().numpy().copy() for p in model.parameters()]
        opt.step()
        for r, g, s in zip(ref, grads, st):
            oracle.optim8bit_step(kind, r.reshape(-1), g.reshape(-1), s["s1"], s["s2"], s["a1"], s["a2"], step=t, **hp)
        for p, r in zip(model.parameters(), ref):
            assert np.array_equal(p.detach().cpu().numpy().view(np.uint32), r.view(np.uint32))


def test_state_dict_resume_is_bit_identical(q8):
    m1 = make_model()
    m2 = copy.deepcopy(m1)
    o1 = q8.AdamW8bit(m1.parameters(), lr=2e-3)
    o2 = q8.AdamW8bit(m2.parameters(), lr=2e-3)
    x = torch.randn(32, 300, device=DEV)

    def step(m, o):
        o.zero_grad()
        m(x).square().mean().backward()
        o.step()

    for _ in range(3):
        step(m1, o1)
        step(m2, o2)
    sd = copy.deepcopy(o2.state_dict())
    msd = copy.deepcopy(m2.state_dict())
    m3 = make_model()
    m3.load_state_dict(msd)
    o3 = q8.AdamW8bit(m3.parameters(), lr=2e-3)
    o3.load_state_dict(sd)
    for _ in range(2):
        step(m1, o1)
        step(m3, o3)
    for a, b in zip(m1.parameters(), m3.parameters()):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_zero1_single_rank_equals_plain_step(q8):
    n = 7 * 2048 + 100
    hp = dict(synth.HPARAMS["adamw"])
    zo = q8.Zero1Optimizer8bit(n, kind="adamw", grad_dtype=torch.bfloat16, device=DEV, **hp)
    p = synth.params(n).to(DEV)
    zo.params[:n] = p
    s1, a1 = synth.zero_state(n, device=DEV)
    s2, a2 = synth.zero_state(n, device=DEV)
    for t in range(1, 4):
        g = synth.grads(n, step=t, dtype="bfloat16").to(DEV)
        zo.grads[:n] = g
        zo.step()
        q8.optim8bit_step("adamw", p, g, s1, s2, a1, a2, step=t, **hp)
    torch.cuda.synchronize()
    assert torch.equal(zo.params[:n].view(torch.int32), p.view(torch.int32))
    assert torch.equal(zo.s1[:n], s1) and torch.equal(zo.absmax2[:a2.numel()], a2)


def test_state_bytes_matches_paper_arithmetic(q8):
    # 8 GB of 32-bit Adam state per 1B params -> 2 GB in 8 bits (+ absmax per block)
    assert abs(q8.state_bytes(10**9, "adam") / 1e9 - 2.0039) < 1e-3
    assert abs(q8.state_bytes(10**9, "momentum") / 1e9 - 1.00195) < 1e-4


@pytest.mark.parametrize("kind", ["adam", "adamw", "momentum"])
@pytest.mark.parametrize("gdt", ["float32", "bfloat16"])
def test_32bit_state_step_matches_oracle(q8, kind, gdt):
    """q8_optim32bit_step_multi == the oracle's 32-bit step (pinned to torch.optim), bit for bit."""
    hp = dict(synth.HPARAMS[kind])
    sizes = [1, 2048 * 3 + 7, 100_000]
    ents, refs = [], []
    for i, n in enumerate(sizes):
        p = synth.params(n, seed=i)
        m = synth.params(n, seed=50 + i, std=1e-3)
        r = synth.params(n, seed=90 + i, std=1e-3).abs() ** 2
        ents.append([p.to(DEV), None, m.to(DEV), r.to(DEV) if kind != "momentum" else None])
        refs.append([p.numpy().copy(), m.numpy().copy(), r.numpy().copy()])
    for t in (1, 2):
        gs = [synth.grads(n, step=t, seed=i, dtype=gdt) for i, n in enumerate(sizes)]
        q8.optim32bit_step_multi(kind, [(e[0], g.to(DEV), e[2], e[3]) for e, g in zip(ents, gs)], step=t, **hp)
        for ref, g in zip(refs, gs):
            oracle.optim32bit_step(kind, ref[0], synth.to_f32_numpy(g), ref[1],
                                   ref[2] if kind != "momentum" else None, step=t, **hp)
    torch.cuda.synchronize()
    for e, ref in zip(ents, refs):
        assert np.array_equal(e[0].cpu().numpy().view(np.uint32), ref[0].view(np.uint32))
        assert np.array_equal(e[2].cpu().numpy().view(np.uint32), ref[1].view(np.uint32))
        if kind != "momentum":
            assert np.array_equal(e[3].cpu().numpy().view(np.uint32), ref[2].view(np.uint32))


def test_stable_embedding_keeps_32bit_states(q8):
    """the embedding layer's states stay 32-bit, the rest 8-bit; both match the oracle."""
    torch.manual_seed(1)
    emb = q8.StableEmbedding(500, 64).to(DEV)
    lin = torch.nn.Linear(64, 40).to(DEV)
    params = list(emb.parameters()) + list(lin.parameters())
    ref = [p.detach().cpu().numpy().copy().reshape(-1) for p in params]
    opt = q8.Adam8bit(params, lr=1e-3)
    st32 = {0: (np.zeros(ref[0].size, np.float32), np.zeros(ref[0].size, np.float32))}
    st8 = {i: [np.zeros(r.size, np.uint8), np.zeros(r.size, np.uint8), np.zeros((r.size + 2047) // 2048, np.float32),
               np.zeros((r.size + 2047) // 2048, np.float32)] for i, r in enumerate(ref) if i > 0}
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, bias_correction=True)
    x = torch.randint(0, 500, (16, 12), device=DEV)
    for t in (1, 2, 3):
        opt.zero_grad()
        lin(emb(x)).square().mean().backward()
        grads = [p.grad.detach().cpu().numpy().copy().reshape(-1) for p in params]
        opt.step()
        oracle.optim32bit_step("adam", ref[0], grads[0], st32[0][0], st32[0][1], step=t, **hp)
        for i in st8:
            s1, s2, a1, a2 = st8[i]
            oracle.optim8bit_step("adam", ref[i], grads[i], s1, s2, a1, a2, step=t, **hp)
    assert "m" in opt.state[emb.weight] and "s1" not in opt.state[emb.weight]
    assert "s1" in opt.state[lin.weight]
    for p, r in zip(params, ref):
        assert np.array_equal(p.detach().cpu().numpy().reshape(-1).view(np.uint32), r.view(np.uint32))


def test_cached_descriptors_follow_new_storage(q8):
    # the descriptor cache refreshes gradient pointers each step; a parameter whose .data is
    # re-pointed between steps must be stepped in its new storage (and the old one left alone)
    model = make_model()
    opt = q8.AdamW8bit(model.parameters(), lr=1e-3)
    x = torch.randn(16, 300, device=DEV)
    ref = [p.detach().cpu().numpy().copy() for p in model.parameters()]
    st = [dict(s1=np.zeros(p.size, np.uint8), s2=np.zeros(p.size, np.uint8),
               a1=np.zeros((p.size + 2047) // 2048, np.float32), a2=np.zeros((p.size + 2047) // 2048, np.float32))
          for p in ref]
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, bias_correction=True)  # AdamW8bit defaults
    old = None
    for t in range(1, 4):
        if t == 3:
            p0 = next(model.parameters())
            old = p0.data
            p0.data = p0.data.clone()
            old_copy = old.clone()
        opt.zero_grad()
        model(x).square().mean().backward()
        grads = [p.grad.detach().cpu().numpy().copy() for p in model.parameters()]
        opt.step()
        for r, g, s in zip(ref, grads, st):
            oracle.optim8bit_step("adamw", r.reshape(-1), g.reshape(-1), s["s1"], s["s2"], s["a1"], s["a2"], step=t, **hp)
    torch.cuda.synchronize()
    for p, r in zip(model.parameters(), ref):
        assert np.array_equal(p.detach().cpu().numpy().view(np.uint32), r.view(np.uint32))
    assert torch.equal(old, old_copy)  # the abandoned storage was not written
