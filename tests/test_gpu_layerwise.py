"""GPU parity of the layer-wise 8-bit optimizers (8-bit LAMB / LARS, T5 P:366-367; readings L1-L4)
through the C ABI (q8_optim8bit_step_layerwise) against the oracle, tensor by tensor.

Every output is compared bit for bit: the per-tensor scales RN(lr * ratio), the parameters, the
codes and the absmax values.  The norms are binary64 sums in different orders on the two sides
(L3), so the scales could in principle differ in their last bit; with the seeded inputs below
they are identical, and given identical scales every other output is a unique function of the
inputs (as for the element-wise step)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"
LAMB = dict(synth.HPARAMS["lamb"])
LARS = dict(synth.HPARAMS["lars"])
ETA = LARS.pop("trust_coefficient")
HP = {"lamb": LAMB, "lars": LARS}


@pytest.fixture(scope="module")
def q8():
    import paper_2110_02861_b200 as m
    return m


def _make(kind, sizes, gdt, seed0=0):
    two = kind == "lamb"
    ents, refs = [], []
    for i, n in enumerate(sizes):
        p = synth.params(n, seed=seed0 + i)
        s1, a1 = synth.random_state(n, seed=seed0 + 100 + i, scale=1e-3)
        s2, a2 = synth.random_state(n, seed=seed0 + 200 + i, scale=1e-6)
        ents.append([p.to(DEV), None, s1.to(DEV), s2.to(DEV) if two else None, a1.to(DEV), a2.to(DEV) if two else None])
        refs.append([p.numpy().copy(), s1.numpy().copy(), s2.numpy().copy(), a1.numpy().copy(), a2.numpy().copy()])
    return ents, refs


def _step_both(q8, kind, ents, refs, sizes, gdt, t, hp, teacher_force=False):
    """One GPU step and one oracle step per tensor.  teacher_force: the oracle first computes its own
    scale on a copy (returned as `exp`), then steps the references with the GPU's scale (reading L3:
    the binary64 norm sums may be ordered differently, so the fp32 scale may differ in its last bit;
    given one scale every other output is unique), so every tensor is compared bit for bit."""
    gs = [synth.grads(n, step=t, seed=7 + i, dtype=gdt) for i, n in enumerate(sizes)]
    for e, g in zip(ents, gs):
        e[1] = g.to(DEV)
    scales = q8.optim8bit_step_layerwise(kind, [tuple(e) for e in ents], step=t, trust_coefficient=ETA, **hp)
    torch.cuda.synchronize()
    got = scales.cpu().numpy()
    exp = []
    two = kind == "lamb"
    for i, (r, g) in enumerate(zip(refs, gs)):
        gf = synth.to_f32_numpy(g)
        if teacher_force:
            c = [x.copy() for x in r]
            exp.append(oracle.optim8bit_layerwise_step(kind, c[0], gf, c[1], c[2] if two else None, c[3],
                                                       c[4] if two else None, step=t, trust_coefficient=ETA, **hp))
            oracle.optim8bit_layerwise_step(kind, r[0], gf, r[1], r[2] if two else None, r[3], r[4] if two else None,
                                            step=t, trust_coefficient=ETA, forced_scale=float(got[i]), **hp)
        else:
            exp.append(oracle.optim8bit_layerwise_step(kind, r[0], gf, r[1], r[2] if two else None, r[3],
                                                       r[4] if two else None, step=t, trust_coefficient=ETA, **hp))
    return got, np.array(exp, np.float32)


def _assert_equal(kind, ents, refs):
    for i, (e, r) in enumerate(zip(ents, refs)):
        assert np.array_equal(e[0].cpu().numpy().view(np.uint32), r[0].view(np.uint32)), f"p of tensor {i}"
        assert np.array_equal(e[2].cpu().numpy(), r[1]), f"s1 of tensor {i}"
        assert np.array_equal(e[4].cpu().numpy().view(np.uint32), r[3].view(np.uint32)), f"absmax1 of tensor {i}"
        if kind == "lamb":
            assert np.array_equal(e[3].cpu().numpy(), r[2]), f"s2 of tensor {i}"
            assert np.array_equal(e[5].cpu().numpy().view(np.uint32), r[4].view(np.uint32)), f"absmax2 of tensor {i}"


@pytest.mark.parametrize("kind", ["lamb", "lars"])
@pytest.mark.parametrize("gdt", ["float32", "float16", "bfloat16"])
def test_layerwise_matches_oracle(q8, kind, gdt):
    sizes = [1, 17, 2047, 2049, 3 * 2048 + 5, 100_003, 1 << 20]
    ents, refs = _make(kind, sizes, gdt)
    for t in (1, 2, 3):
        got, exp = _step_both(q8, kind, ents, refs, sizes, gdt, t, HP[kind])
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), (t, got, exp)
    _assert_equal(kind, ents, refs)


@pytest.mark.parametrize("kind", ["lamb", "lars"])
def test_layerwise_hparam_variants(q8, kind):
    sizes = [5000, 70_001]
    variants = ([dict(LAMB, weight_decay=0.0), dict(LAMB, bias_correction=False), dict(LAMB, lr=0.02, beta2=0.99)]
                if kind == "lamb" else [dict(LARS, weight_decay=0.0), dict(LARS, beta1=0.0), dict(LARS, lr=1.0)])
    for j, hp in enumerate(variants):
        ents, refs = _make(kind, sizes, "bfloat16", seed0=10 * j)
        for t in (1, 4):
            got, exp = _step_both(q8, kind, ents, refs, sizes, "bfloat16", t, hp)
            assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
        _assert_equal(kind, ents, refs)


@pytest.mark.parametrize("kind", ["lamb", "lars"])
def test_layerwise_zero_tensors_and_empty(q8, kind):
    """A zero weight tensor (trust ratio falls back to 1, L1/L2) and empty tensors (scale = lr)."""
    sizes = [4096, 0, 3000, 0]
    ents, refs = _make(kind, sizes, "float32")
    ents[0][0].zero_()
    refs[0][0][:] = 0
    got, exp = _step_both(q8, kind, ents, refs, sizes, "float32", 1, HP[kind])
    assert got[1] == np.float32(HP[kind]["lr"]) and got[3] == np.float32(HP[kind]["lr"])
    assert got[0] == exp[0] and got[2] == exp[2]
    _assert_equal(kind, ents, refs)


@pytest.mark.parametrize("gdt", ["float32", "bfloat16"])
def test_lamb_norm_segments_span_blocks_and_tensors(q8, gdt):
    """LAMB's norms pass keeps running sums over a sub-block's consecutive blocks of one tensor and
    reduces once per segment (DESIGN 6.10): ~3,400 blocks give every sub-block several blocks, with
    ranges that start and end inside tensors and cross short tensors.  Scales within 1 fp32 ulp (L3),
    then teacher-forced: every output bit for bit."""
    sizes = [3_000_000, 5, 2_500_007, 2049, 1, 1_500_000, 4095]
    ents, refs = _make("lamb", sizes, gdt, seed0=77)
    for t in (1, 2):
        got, exp = _step_both(q8, "lamb", ents, refs, sizes, gdt, t, HP["lamb"], teacher_force=True)
        ulps = np.abs(got.view(np.int32).astype(np.int64) - exp.view(np.int32).astype(np.int64))
        assert ulps.max() <= 1, (got, exp)
        _assert_equal("lamb", ents, refs)


@pytest.mark.parametrize("kind", ["lars", "lamb"])
def test_layerwise_chunks_over_384_tensors(q8, kind):
    """More tensors than one launch takes: the workspace's partials are reused per chunk."""
    rng = np.random.default_rng(5)
    sizes = [int(x) for x in rng.integers(1, 9000, size=400)]
    ents, refs = _make(kind, sizes, "bfloat16")
    got, exp = _step_both(q8, kind, ents, refs, sizes, "bfloat16", 1, HP[kind], teacher_force=True)
    ulps = np.abs(got.view(np.int32).astype(np.int64) - exp.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1, (got, exp)
    _assert_equal(kind, ents, refs)


@pytest.mark.parametrize("count", [192, 193])
def test_layerwise_descriptor_table_tiers(q8, count):
    """Lists of <= 192 tensors launch with the 192-entry descriptor table, longer ones with the 384-entry
    table (q8_launch.h kSmallMaxT): both sides of the boundary, LAMB and LARS, bit for bit (teacher-forced)."""
    rng = np.random.default_rng(count)
    sizes = [int(x) for x in rng.integers(1, 5000, size=count)]
    for kind in ("lars", "lamb"):
        ents, refs = _make(kind, sizes, "float16", seed0=count)
        got, exp = _step_both(q8, kind, ents, refs, sizes, "float16", 2, HP[kind], teacher_force=True)
        ulps = np.abs(got.view(np.int32).astype(np.int64) - exp.view(np.int32).astype(np.int64))
        assert ulps.max() <= 1, (got, exp)
        _assert_equal(kind, ents, refs)


def test_lars_resnet50_layer_list(q8):
    """LARS's home workload: the 161 ResNet-50 tensors, bf16 grads, 2 steps."""
    sizes = [int(np.prod(s)) for s in synth.resnet50_shapes()]
    ents, refs = _make("lars", sizes, "bfloat16")
    for t in (1, 2):
        got, exp = _step_both(q8, "lars", ents, refs, sizes, "bfloat16", t, LARS)
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    _assert_equal("lars", ents, refs)


@pytest.mark.parametrize("cls,kind", [("LAMB8bit", "lamb"), ("LARS8bit", "lars")])
def test_layerwise_optimizer_api(q8, cls, kind):
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(300, 700), torch.nn.LayerNorm(700), torch.nn.Linear(700, 50)).to(DEV)
    ref = [p.detach().cpu().numpy().copy().reshape(-1) for p in model.parameters()]
    if kind == "lamb":
        opt = q8.LAMB8bit(model.parameters(), lr=2e-3, weight_decay=0.01)
        hp = dict(lr=2e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01, bias_correction=True)
    else:
        opt = q8.LARS8bit(model.parameters(), lr=0.1, momentum=0.9, weight_decay=5e-4, trust_coefficient=0.001)
        hp = dict(lr=0.1, beta1=0.9, beta2=0.0, eps=1e-8, weight_decay=5e-4, bias_correction=False)
    st = [[np.zeros(r.size, np.uint8), np.zeros(r.size, np.uint8), np.zeros((r.size + 2047) // 2048, np.float32),
           np.zeros((r.size + 2047) // 2048, np.float32)] for r in ref]
    x = torch.randn(64, 300, device=DEV)
    for t in (1, 2, 3):
        opt.zero_grad()
        model(x).square().mean().backward()
        grads = [p.grad.detach().cpu().numpy().copy().reshape(-1) for p in model.parameters()]
        opt.step()
        for r, g, s in zip(ref, grads, st):
            oracle.optim8bit_layerwise_step(kind, r, g, s[0], s[1] if kind == "lamb" else None, s[2],
                                            s[3] if kind == "lamb" else None, step=t, trust_coefficient=0.001, **hp)
    for p, r in zip(model.parameters(), ref):
        assert np.array_equal(p.detach().cpu().numpy().reshape(-1).view(np.uint32), r.view(np.uint32))
        assert "trust_scale" in opt.state[p]


@pytest.mark.parametrize("i", range(8))
def test_layerwise_random_sweep(q8, i):
    # seeded random layer lists and hyper-parameters; the per-tensor scales come from binary64 norms
    # summed in different orders (L3), so they are asserted within one fp32 ulp of the oracle's own,
    # and the oracle is then teacher-forced with the GPU's scales: EVERY tensor matches bit for bit
    rng = np.random.default_rng(700 + i)
    kind = ["lamb", "lars"][i % 2]
    gdt = ["float32", "float16", "bfloat16"][i % 3]
    sizes = [int(rng.integers(1, 40_000)) for _ in range(int(rng.integers(2, 30)))]
    hp = dict(HP[kind])
    hp.update(lr=float(10 ** rng.uniform(-4, -1)), weight_decay=float(rng.choice([0.0, 1e-4, 0.01])))
    if kind == "lamb":
        hp.update(beta2=float(rng.choice([0.99, 0.999])), bias_correction=bool(rng.integers(0, 2)))
    ents, refs = _make(kind, sizes, gdt, seed0=1000 * i)
    t = int(rng.integers(1, 20))
    for _ in range(2):  # two steps: the second starts from teacher-forced (identical) states
        got, exp = _step_both(q8, kind, ents, refs, sizes, gdt, t, hp, teacher_force=True)
        ulps = np.abs(got.view(np.int32).astype(np.int64) - exp.view(np.int32).astype(np.int64))
        assert ulps.max() <= 1, (got, exp)
        _assert_equal(kind, ents, refs)
        t += 1


def test_lars_one_launch_variant():
    """The one-launch LARS (Q8_LARS_ONE_LAUNCH=1: norms, grid barrier, scales, grid barrier, step in one
    cooperative kernel) passes the same teacher-forced parity tests as the default three launches."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, Q8_LARS_ONE_LAUNCH="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", os.path.abspath(__file__),
                        "-k", "lars and not one_launch"], capture_output=True, text=True, env=env, cwd=root,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_lars_workspace_counters_return_to_zero(q8):
    """The LARS norms pass counts every tensor's blocks in the workspace (q8.h: the workspace must be zero-filled
    before its first use and every call leaves it so): after each of several calls -- chunked launches, empty
    tensors, tensors of one and of many blocks -- the counter region is zero again."""
    sizes = [0, 5, 2048, 4096 + 17, 70_000, 0, 3] * 60   # 420 tensors: two launch chunks
    ents, _ = _make("lars", sizes, "float16", seed0=50)
    for i, (e, n) in enumerate(zip(ents, sizes)):
        e[1] = synth.grads(n, step=1, seed=9 + i, dtype="float16").to(DEV)
    tl = q8.TensorList([tuple(e) for e in ents], "lars")
    need = q8.layerwise_workspace_bytes(tl)
    ws = torch.zeros(need, dtype=torch.uint8, device=DEV)
    first = None
    for t in (1, 2, 3):
        scales = q8.optim8bit_step_layerwise("lars", tl, step=t, trust_coefficient=ETA, workspace=ws, **LARS).clone()
        torch.cuda.synchronize()
        counters = ws[:4 * 384]
        assert int(counters.count_nonzero()) == 0, f"call {t}: block counters not reset"
        if first is None:
            first = scales
    # every tensor got a finite scale; empty ones lr (q8.h)
    sc = first.cpu().numpy()
    assert np.all(np.isfinite(sc))
    assert np.all(sc[[i for i, n in enumerate(sizes) if n == 0]] == np.float32(LARS["lr"]))


def test_lars_workspace_reused_across_tensor_lists(q8):
    """One workspace serves a long list and then a short one (an optimizer with several parameter groups):
    the counters sit at a fixed offset (q8.h), so the short list's step is bit-exact against the oracle
    (teacher-forced with the GPU's scales, each within one fp32 ulp of the oracle's own, reading L3)."""
    sizes_a = [70_000, 5, 2048, 300_000, 17] * 20
    sizes_b = [4096 + 1, 9, 50_000]
    ea, _ = _make("lars", sizes_a, "bfloat16", seed0=300)
    eb, rb = _make("lars", sizes_b, "bfloat16", seed0=400)
    for i, (e, n) in enumerate(zip(ea, sizes_a)):
        e[1] = synth.grads(n, step=1, seed=5 + i, dtype="bfloat16").to(DEV)
    ws = torch.zeros(q8.layerwise_workspace_bytes([tuple(e) for e in ea]), dtype=torch.uint8, device=DEV)
    q8.optim8bit_step_layerwise("lars", [tuple(e) for e in ea], step=1, trust_coefficient=ETA, workspace=ws, **LARS)
    gs = [synth.grads(n, step=2, seed=50 + i, dtype="bfloat16") for i, n in enumerate(sizes_b)]
    for e, g in zip(eb, gs):
        e[1] = g.to(DEV)
    got = q8.optim8bit_step_layerwise("lars", [tuple(e) for e in eb], step=2, trust_coefficient=ETA, workspace=ws,
                                      **LARS).cpu().numpy()
    torch.cuda.synchronize()
    for i, (r, g) in enumerate(zip(rb, gs)):
        gf = synth.to_f32_numpy(g)
        c = [x.copy() for x in r]
        exp = oracle.optim8bit_layerwise_step("lars", c[0], gf, c[1], None, c[3], None, step=2,
                                              trust_coefficient=ETA, **LARS)
        assert abs(float(got[i]) - float(exp)) <= float(np.spacing(np.float32(exp))), f"scale {i}"
        oracle.optim8bit_layerwise_step("lars", r[0], gf, r[1], None, r[3], None, step=2, trust_coefficient=ETA,
                                        forced_scale=float(got[i]), **LARS)
    _assert_equal("lars", eb, rb)
