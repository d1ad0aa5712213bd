"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE north_star): codes and absmax bit-exact for a given fp32
pre-quantization input; updated params within 1e-6 max relative error -- with the
pinned fp32 op order (G9) they are expected, and asserted, to be bit-identical.
All inputs come from synth (seeded); every expected value comes from oracle/."""
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


def bits(a):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return a.view(np.uint32) if a.dtype == np.float32 else a


def assert_same(gpu, ref, what):
    g = bits(gpu)
    r = bits(ref)
    if not np.array_equal(g, r):
        idx = np.nonzero(g != r)[0]
        raise AssertionError(f"{what}: {idx.size} mismatches, first at {idx[:8]}: gpu {g[idx[:4]]} ref {r[idx[:4]]}")


# ----------------------------------------------------------------------------- codec

SIZES = [1, 15, 16, 17, 2047, 2048, 2049, 3 * 2048 + 5, 1_000_000, 1 << 20]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("signed", [True, False])
def test_quantize_dequantize_bit_exact(q8, n, signed):
    Q = oracle.dynamic_codebook(signed)
    x = synth.params(n, seed=n, std=1.0)
    if not signed:
        x = x * x
    if n > 4096:  # an all-zero block and an outlier block
        x[2048:4096] = 0
        x[5000] = 1e4
    code_dev = torch.from_numpy(Q).to(DEV)
    a_g, c_g = q8.quantize_blockwise(code_dev, x.to(DEV))
    a_r, c_r = oracle.quantize_blockwise(Q, x.numpy())
    assert_same(a_g, a_r, "absmax")
    assert_same(c_g, c_r, "codes")
    d_g = q8.dequantize_blockwise(code_dev, c_g, a_g)
    assert_same(d_g, oracle.dequantize_blockwise(Q, c_r, a_r), "dequantized")
    a_d, c_d = q8.quantize_blockwise_dynamic(signed, x.to(DEV))
    assert_same(a_d, a_r, "absmax (dynamic)")
    assert_same(c_d, c_r, "codes (dynamic)")


def test_quantize_dynamic_unsigned_negative_inputs(q8):
    """Unsigned table, negative inputs: the nearest code is Q_u[0] = 0 (Eq.3)."""
    Q = oracle.dynamic_codebook(False)
    x = synth.params(3 * 2048 + 11, seed=5, std=1.0)
    a_r, c_r = oracle.quantize_blockwise(Q, x.numpy())
    a_d, c_d = q8.quantize_blockwise_dynamic(False, x.to(DEV))
    assert_same(a_d, a_r, "absmax")
    assert_same(c_d, c_r, "codes")


def _boundaries(Q):
    """Smallest fp32 y (as a float64 value) with oracle code k+1, for k = 0..254: found by
    bisection over fp32 bit patterns with oracle.nearest_code (monotone in y)."""
    def key_to_f(k):  # monotone int -> float32: k >= 0 -> bits k; k < 0 -> -(|bits| + 1)
        u = k if k >= 0 else (0x80000000 | (-k - 1))
        return np.array([u], np.uint32).view(np.float32)[0]

    def code(k):
        return int(oracle.nearest_code(Q, np.float32(key_to_f(k)))[0])

    lo_key, hi_key = -0x3f800001, 0x3f800000  # keys of -1.0 and +1.0
    out = []
    for target in range(1, 256):
        lo, hi = lo_key, hi_key + 1
        while lo < hi:
            mid = (lo + hi) // 2
            if code(mid) >= target:
                hi = mid
            else:
                lo = mid + 1
        out.append(float(key_to_f(lo)) if lo <= hi_key else np.inf)
    return np.array(out, np.float64)


@pytest.mark.slow
@pytest.mark.parametrize("path", ["generic", "dynamic"])
@pytest.mark.parametrize("signed", [True, False])
def test_nearest_code_exhaustive_fp32(q8, signed, path):
    """Every finite fp32 y in [-1, 1] (signed) / [0, 1] (unsigned) through the public
    quantize_blockwise (generic table: Eytzinger 8-step search) and quantize_blockwise_dynamic
    (built-in table: the step kernel's bucketed search): one +1.0 per 2048-block makes
    N_b = 1, so y/N_b = y exactly and the codes are the nearest codes.  Expected: the
    oracle's step function, evaluated with torch.searchsorted over its 255 decision
    boundaries."""
    Q = oracle.dynamic_codebook(signed)
    bnd = torch.from_numpy(_boundaries(Q)).to(DEV)
    code_dev = torch.from_numpy(Q).to(DEV)
    ranges = [(0, 0x3f800000 + 1)]  # +0 .. +1.0
    if signed:
        ranges.append((0x80000000, 0xbf800000 + 1))  # -0 .. -1.0
    chunk = 2047 * (1 << 16)
    total = 0
    for lo, hi in ranges:
        for s in range(lo, hi, chunk):
            e = min(s + chunk, hi)
            k = torch.arange(s, e, dtype=torch.int64, device=DEV)
            y = torch.where(k >= 2 ** 31, k - 2 ** 32, k).to(torch.int32).view(torch.float32)
            nb = (y.numel() + 2046) // 2047
            x = torch.ones(nb * 2048, dtype=torch.float32, device=DEV)
            xv = x.view(nb, 2048)
            flat = torch.zeros(nb * 2047, dtype=torch.float32, device=DEV)
            flat[:y.numel()] = y
            xv[:, 1:] = flat.view(nb, 2047)
            if path == "generic":
                a, c = q8.quantize_blockwise(code_dev, x)
            else:
                a, c = q8.quantize_blockwise_dynamic(signed, x)
            assert torch.all(a == 1.0)
            got = c.view(nb, 2048)[:, 1:].reshape(-1)[:y.numel()].to(torch.int64)
            exp = torch.searchsorted(bnd, y.to(torch.float64), right=True)
            bad = torch.nonzero(got != exp)
            assert bad.numel() == 0, (signed, s, bad[:5].flatten().tolist())
            total += y.numel()
    assert total == (0x3f800001 * (2 if signed else 1))


# ----------------------------------------------------------------------------- step

KINDS = ["adam", "adamw", "momentum"]
GDTS = ["float32", "float16", "bfloat16"]


def make_case(n, kind, gdt, seed, random_state):
    p = synth.params(n, seed=seed)
    if random_state:
        s1, a1 = synth.random_state(n, seed=seed + 1, scale=1e-3)
        s2, a2 = synth.random_state(n, seed=seed + 2, scale=1e-6)
    else:
        s1, a1 = synth.zero_state(n)
        s2, a2 = synth.zero_state(n)
    return p, s1, a1, s2, a2


def run_both(q8, kind, gdt, n, steps, hp, seed=0, random_state=False, outliers=0.0, first_step=1):
    p, s1, a1, s2, a2 = make_case(n, kind, gdt, seed, random_state)
    gp = [t.to(DEV).clone() for t in (p, s1, a1, s2, a2)]
    cp = [t.numpy().copy() for t in (p, s1, a1, s2, a2)]
    for t in range(first_step, first_step + steps):
        g = synth.grads(n, step=t, seed=seed, dtype=gdt, outlier_frac=outliers)
        q8.optim8bit_step(kind, gp[0], g.to(DEV), gp[1], gp[3], gp[2], gp[4], step=t, **hp)
        oracle.optim8bit_step(kind, cp[0], synth.to_f32_numpy(g), cp[1], cp[3], cp[2], cp[4], step=t, nthreads=8,
                              **hp)
    torch.cuda.synchronize()
    return gp, cp


def check(gp, cp, kind, what=""):
    assert_same(gp[0], cp[0], f"{what} p")
    assert_same(gp[1], cp[1], f"{what} s1")
    assert_same(gp[2], cp[2], f"{what} absmax1")
    if kind != "momentum":
        assert_same(gp[3], cp[3], f"{what} s2")
        assert_same(gp[4], cp[4], f"{what} absmax2")


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gdt", GDTS)
@pytest.mark.parametrize("n", [1, 17, 2048, 3 * 2048 + 5, 100_003])
def test_step_single_bit_exact(q8, kind, gdt, n):
    hp = dict(synth.HPARAMS[kind])
    for random_state in (False, True):
        gp, cp = run_both(q8, kind, gdt, n, 1, hp, seed=n, random_state=random_state, first_step=3)
        check(gp, cp, kind, f"rs={random_state}")


@pytest.mark.parametrize("kind", ["adam", "adamw"])
@pytest.mark.parametrize("bc", [True, False])
@pytest.mark.parametrize("wd", [0.0, 0.05])
def test_step_hparam_variants(q8, kind, bc, wd):
    hp = dict(synth.HPARAMS["adam_paper"])
    hp.update(bias_correction=bc, weight_decay=wd)
    gp, cp = run_both(q8, kind, "bfloat16", 5 * 2048 + 77, 3, hp, seed=9, random_state=True)
    check(gp, cp, kind)


@pytest.mark.parametrize("kind,gdt", [("adam", "float32"), ("adamw", "bfloat16"), ("momentum", "float16")])
def test_ten_steps_config1_free_running(q8, kind, gdt):
    """BASELINE config 1: 10 steps on one flat 1M-element tensor, free running, bit-exact."""
    hp = dict(synth.HPARAMS[kind])
    gp, cp = run_both(q8, kind, gdt, 1 << 20, 10, hp, seed=1)
    check(gp, cp, kind, "10 steps")


def test_outliers_and_tiny_states(q8):
    """Gradient spikes x100 and tiny second moments (exercise the IEEE-division
    normalize path for N_b < 2^-70 and the zero-absmax path)."""
    hp = dict(synth.HPARAMS["adam"])
    gp, cp = run_both(q8, "adam", "float32", 64 * 2048 + 3, 3, hp, seed=4, outliers=1e-3)
    check(gp, cp, "adam", "outliers")
    n = 8 * 2048
    p = synth.params(n)
    g = torch.zeros(n)
    g[:2048] = 1e-30   # r ~ 1e-63 underflows to 0; m ~ 1e-31 -> slow-division path
    g[2048:4096] = 1e-20
    g[4096:6144] = 3e-24
    s1, a1 = synth.zero_state(n)
    s2, a2 = synth.zero_state(n)
    gp = [t.to(DEV) for t in (p, s1, a1, s2, a2)]
    cp = [t.numpy().copy() for t in (p, s1, a1, s2, a2)]
    q8.optim8bit_step("adam", gp[0], g.to(DEV), gp[1], gp[3], gp[2], gp[4], step=1, **hp)
    oracle.optim8bit_step("adam", cp[0], g.numpy(), cp[1], cp[3], cp[2], cp[4], step=1, **hp)
    check(gp, cp, "adam", "tiny")


@pytest.mark.parametrize("gdt", ["float16"])
def test_multi_tensor_resnet50(q8, gdt):
    """BASELINE config 3: 8-bit Momentum over the ResNet-50 tensor list in one multi-tensor
    launch == per-tensor oracle steps (blocks are per tensor)."""
    hp = dict(synth.HPARAMS["momentum"])
    shapes = synth.resnet50_shapes()
    ents, refs = [], []
    for i, sh in enumerate(shapes):
        n = synth.numel(sh)
        p = synth.params(n, seed=100 + i)
        g = synth.grads(n, step=1, seed=100 + i, dtype=gdt)
        s1, a1 = synth.random_state(n, seed=200 + i)
        ents.append((p.to(DEV), g.to(DEV), s1.to(DEV), None, a1.to(DEV), None))
        refs.append((p.numpy().copy(), synth.to_f32_numpy(g), s1.numpy().copy(), a1.numpy().copy()))
    tl = q8.TensorList(ents)
    q8.optim8bit_step_multi("momentum", tl, step=2, **hp)
    torch.cuda.synchronize()
    for i, (e, r) in enumerate(zip(ents, refs)):
        p, g, s1, a1 = r
        oracle.optim8bit_step("momentum", p, g, s1, None, a1, None, step=2, **hp)
        assert_same(e[0], p, f"t{i} p")
        assert_same(e[2], s1, f"t{i} s1")
        assert_same(e[4], a1, f"t{i} a1")


def test_multi_tensor_many_launches_and_empty(q8):
    """> 384 tensors (several launches), empty tensors skipped, Adam with two states."""
    hp = dict(synth.HPARAMS["adam"])
    sizes = [0, 5, 2048, 3000, 1] * 90  # 450 entries
    ents, refs = [], []
    for i, n in enumerate(sizes):
        p = synth.params(n, seed=i)
        g = synth.grads(n, step=1, seed=i, dtype="bfloat16")
        s1, a1 = synth.random_state(n, seed=i)
        s2, a2 = synth.random_state(n, seed=i + 7, scale=1e-6)
        ents.append(tuple(t.to(DEV) for t in (p, g, s1, s2, a1, a2)))
        refs.append([t.numpy().copy() for t in (p, s1, s2, a1, a2)] + [synth.to_f32_numpy(g)])
    q8.optim8bit_step_multi("adam", ents, step=4, **hp)
    torch.cuda.synchronize()
    for i, (e, r) in enumerate(zip(ents, refs)):
        p, s1, s2, a1, a2, g = r
        if p.size:
            oracle.optim8bit_step("adam", p, g, s1, s2, a1, a2, step=4, **hp)
        for k, (gt, rt) in enumerate(zip((e[0], e[2], e[3], e[4], e[5]), (p, s1, s2, a1, a2))):
            assert_same(gt, rt, f"t{i}.{k}")


def test_eytzinger_step_variant_bit_exact():
    """The pure 8-step Eytzinger search variant of the step kernel (Q8_SEARCH=eytzinger)
    passes the same single-step parity cases (separate process: the variant is chosen once
    per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, Q8_SEARCH="eytzinger")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", __file__, "-k",
                        "test_step_single_bit_exact or test_ten_steps or test_multi_tensor_resnet50"],
                       env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_errors_surface_as_exceptions(q8):
    p = torch.zeros(4099, device=DEV)
    g = torch.zeros(4099, device=DEV)
    s = torch.zeros(4099, dtype=torch.uint8, device=DEV)
    a = torch.zeros(3, device=DEV)
    with pytest.raises(q8.Q8Error):
        q8.optim8bit_step("adam", p[1:], g[1:], s[1:], s[1:], a, a, lr=1e-3, step=1)  # misaligned p
    with pytest.raises(q8.Q8Error):
        q8.optim8bit_step("adam", p, g, s, s, a, a, lr=1e-3, step=1, blocksize=4096)


@pytest.mark.parametrize("n", [1, 17, 2049, 3 * 2048 + 5, 1_000_000])
@pytest.mark.parametrize("table", ["dynamic_signed", "linear_signed", "linear_unsigned"])
def test_tensorwise_codec_bit_exact(q8, n, table):
    """Eq.3: one absmax for the whole tensor (oracle: block size = n)."""
    Q = {"dynamic_signed": oracle.dynamic_codebook(True), "linear_signed": oracle.linear_codebook(True),
         "linear_unsigned": oracle.linear_codebook(False)}[table]
    x = synth.params(n, seed=n + 3, std=1.0)
    if table == "linear_unsigned":
        x = x.abs()
    if n > 10:
        x[n // 2] = 37.0  # an outlier dominates the single normalization constant
    code_dev = torch.from_numpy(Q).to(DEV)
    a_g, c_g = q8.quantize_tensorwise(code_dev, x.to(DEV))
    a_r, c_r = oracle.quantize_blockwise(Q, x.numpy(), blocksize=n)
    assert_same(a_g, a_r, "absmax")
    assert_same(c_g, c_r, "codes")
    assert_same(q8.dequantize_tensorwise(code_dev, c_g, a_g), oracle.dequantize_blockwise(Q, c_r, a_r, n), "deq")


@pytest.mark.parametrize("signed", [True, False])
def test_linear_type_zero_round_trip(q8, signed):
    """Reading L0: exact zeros in a block with a nonzero absmax come back as exact zeros through the
    linear type (block-wise and tensor-wise codecs), identically to the oracle."""
    n = 3 * 2048 + 77
    Q = oracle.linear_codebook(signed)
    x = synth.params(n, seed=41, std=1.0)
    if not signed:
        x = x.abs()
    x[::3] = 0.0
    code_dev = torch.from_numpy(Q).to(DEV)
    a_g, c_g = q8.quantize_blockwise(code_dev, x.to(DEV))
    a_r, c_r = oracle.quantize_blockwise(Q, x.numpy())
    assert_same(a_g, a_r, "absmax")
    assert_same(c_g, c_r, "codes")
    d = q8.dequantize_blockwise(code_dev, c_g, a_g).cpu()
    assert torch.all(d[::3] == 0.0) and torch.all(c_g.cpu()[::3] == (127 if signed else 0))
    a_t, c_t = q8.quantize_tensorwise(code_dev, x.to(DEV))
    assert torch.all(q8.dequantize_tensorwise(code_dev, c_t, a_t).cpu()[::3] == 0.0)


# Ragged last blocks of multi-tensor launches ("n/B blocks" per tensor): tails of 5 .. 2032
# elements, multiples of 16 and not, single-block tensors and tensors of several blocks, so one
# sub-block's contiguous block range alternates tails (guarded direct loads) and full blocks (TMA stage);
# two steps, every tensor bit for bit.
TAIL_SIZES = [16, 2048 + 16, 48, 5, 2048 * 3 + 2032, 1024, 17, 2048 + 1008, 4096, 2048 + 1000, 64, 2048 * 2 + 32]


@pytest.mark.parametrize("kind,gdt", [("momentum", "float16"), ("adam", "bfloat16"), ("adamw", "float32"),
                                      ("momentum", "float32")])
def test_multi_tensor_staged_tails(q8, kind, gdt):
    hp = dict(synth.HPARAMS[kind])
    two = kind != "momentum"
    sizes = TAIL_SIZES * 6
    ents, refs = [], []
    for i, n in enumerate(sizes):
        p = synth.params(n, seed=300 + i)
        g = synth.grads(n, step=1, seed=300 + i, dtype=gdt)
        s1, a1 = synth.random_state(n, seed=400 + i)
        s2, a2 = synth.random_state(n, seed=500 + i, scale=1e-6)
        ents.append((p.to(DEV), g.to(DEV), s1.to(DEV), s2.to(DEV) if two else None, a1.to(DEV),
                     a2.to(DEV) if two else None))
        refs.append([t.numpy().copy() for t in (p, s1, s2, a1, a2)] + [synth.to_f32_numpy(g)])
    for t in (3, 4):
        q8.optim8bit_step_multi(kind, ents, step=t, **hp)
        for r in refs:
            p, s1, s2, a1, a2, g = r
            oracle.optim8bit_step(kind, p, g, s1, s2 if two else None, a1, a2 if two else None, step=t, **hp)
    torch.cuda.synchronize()
    for i, (e, r) in enumerate(zip(ents, refs)):
        assert_same(e[0], r[0], f"t{i} p")
        assert_same(e[2], r[1], f"t{i} s1")
        assert_same(e[4], r[3], f"t{i} a1")
        if two:
            assert_same(e[3], r[2], f"t{i} s2")
            assert_same(e[5], r[4], f"t{i} a2")
