"""Pins for the oracle's layer-wise optimizers, 8-bit LAMB and LARS (T5; readings L1-L4
in oracle.c / DESIGN.md 3).  The paper prints no formula for them, so the pins hold the oracle to
the textbook algorithms through routes that do not retype its fp32 code:

* LAMB's states equal the (torch-pinned) Adam oracle's states bit for bit; its parameter update
  matches the UNFOLDED textbook form of You et al. 2020 Alg. 2 evaluated in float64 from those
  states; the trust ratio makes |w' - w| = lr |w| (closed form), a 1-element tensor moves by
  exactly lr |w|, and a zero tensor falls back to ratio 1.
* LARS equals torch.optim.SGD(lr=1, momentum=beta) fed the trust-scaled gradient
  RN(a * RN(g + RN(wd * w))), with a = RN(lr * eta |w| / (|g| + wd |w|)) from numpy norms; with
  zero state and wd = 0 the first step moves w by exactly lr * eta * |w|.
* The 8-bit steps equal dequantize -> 32-bit step -> block quantization (bit-exact) and track the
  32-bit steps within quantization error."""
import numpy as np
import pytest
import torch

import oracle
import synth

LAMB = dict(synth.HPARAMS["lamb"])
LARS = dict(synth.HPARAMS["lars"])
ETA = LARS.pop("trust_coefficient")


def _state(n, seed, std):
    return synth.params(n, seed=seed, std=std).numpy()


def test_lamb_states_equal_adam_states():
    n = 3 * 2048 + 77
    p = synth.params(n).numpy()
    g = synth.grads(n, step=2).numpy()
    m0, r0 = _state(n, 11, 1e-3), np.abs(_state(n, 12, 1e-3)) ** 2
    ml, rl, ma, ra = m0.copy(), r0.copy(), m0.copy(), r0.copy()
    oracle.optim32bit_layerwise_step("lamb", p.copy(), g, ml, rl, step=2, **LAMB)
    adam = dict(LAMB, weight_decay=0.0)
    oracle.optim32bit_step("adam", p.copy(), g, ma, ra, step=2, **adam)
    assert np.array_equal(ml.view(np.uint32), ma.view(np.uint32))
    assert np.array_equal(rl.view(np.uint32), ra.view(np.uint32))


@pytest.mark.parametrize("wd,bc,step", [(0.01, True, 3), (0.0, True, 1), (0.1, False, 5)])
def test_lamb_matches_unfolded_textbook_form(wd, bc, step):
    h = dict(LAMB, weight_decay=wd, bias_correction=bc, lr=0.05)
    n = 5000
    p0 = synth.params(n, seed=3).numpy()
    g = synth.grads(n, step=step).numpy()
    m, r = _state(n, 21, 1e-3), np.abs(_state(n, 22, 1e-3)) ** 2
    p = p0.copy()
    a = oracle.optim32bit_layerwise_step("lamb", p, g, m, r, step=step, **h)
    # You et al. 2020 Alg. 2 in float64 from the (Adam-pinned) new states m, r
    b1, b2 = h["beta1"], h["beta2"]
    m64, r64, w = m.astype(np.float64), r.astype(np.float64), p0.astype(np.float64)
    mh = m64 / (1 - b1 ** step) if bc else m64
    vh = r64 / (1 - b2 ** step) if bc else r64
    u = mh / (np.sqrt(vh) + h["eps"]) + wd * w
    ratio = np.linalg.norm(w) / np.linalg.norm(u)
    assert a == pytest.approx(h["lr"] * ratio, rel=1e-6)
    expect = w - h["lr"] * ratio * u
    np.testing.assert_allclose(p, expect, rtol=0, atol=4 * np.spacing(np.abs(p0)).max())
    # trust ratio: the update has norm lr * |w|
    assert np.linalg.norm(p.astype(np.float64) - w) == pytest.approx(h["lr"] * np.linalg.norm(w), rel=1e-4)


def test_lamb_single_element_closed_form():
    for w0, gv in ((0.5, 0.3), (-2.0, 0.7), (0.25, -1.0)):
        p = np.array([w0], np.float32)
        a = oracle.optim32bit_layerwise_step("lamb", p, np.array([gv], np.float32), np.zeros(1, np.float32),
                                             np.zeros(1, np.float32), step=1, **dict(LAMB, weight_decay=0.0, lr=0.1))
        # u = sign(g) * (something > 0); ratio = |w|/|u|  ->  w' = w - lr |w| sign(g)
        assert p[0] == pytest.approx(w0 - 0.1 * abs(w0) * np.sign(gv), rel=1e-6)
        assert a > 0


def test_lamb_zero_weights_use_unit_ratio():
    n = 100
    p = np.zeros(n, np.float32)
    g = synth.grads(n, step=1).numpy()
    a = oracle.optim32bit_layerwise_step("lamb", p, g, np.zeros(n, np.float32), np.zeros(n, np.float32), step=1,
                                         **LAMB)
    assert a == np.float32(LAMB["lr"])
    # t = 1 from zero state: u = g / (|g| + eps) (closed form of bias-corrected Adam), w' = -lr u
    expect = -LAMB["lr"] * g.astype(np.float64) / (np.abs(g.astype(np.float64)) + LAMB["eps"])
    np.testing.assert_allclose(p, expect, rtol=1e-5)


def _lars_torch(p0, m0, g, a, wd, beta):
    gp = (np.float32(a) * (g + np.float32(wd) * p0).astype(np.float32)).astype(np.float32)
    w = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.SGD([w], lr=1.0, momentum=beta, dampening=0, foreach=False)
    opt.state[w]["momentum_buffer"] = torch.from_numpy(m0.copy())
    w.grad = torch.from_numpy(gp)
    opt.step()
    return w.detach().numpy(), opt.state[w]["momentum_buffer"].numpy()


@pytest.mark.parametrize("wd", [5e-4, 0.0])
def test_lars_equals_sgd_on_trust_scaled_gradient(wd):
    h = dict(LARS, weight_decay=wd)
    n = 3 * 2048 + 5
    p0 = synth.params(n, seed=5).numpy()
    g = synth.grads(n, step=4).numpy()
    m0 = _state(n, 31, 1e-3)
    w64, g64 = p0.astype(np.float64), g.astype(np.float64)
    a_np = np.float32(h["lr"] * ETA * np.linalg.norm(w64) / (np.linalg.norm(g64) + wd * np.linalg.norm(w64)))
    p, m = p0.copy(), m0.copy()
    a = oracle.optim32bit_layerwise_step("lars", p, g, m, None, step=4, trust_coefficient=ETA, **h)
    assert abs(int(a.view(np.int32)) - int(a_np.view(np.int32))) <= 1
    tp, tm = _lars_torch(p0, m0, g, a, wd, h["beta1"])
    assert np.array_equal(m.view(np.uint32), tm.view(np.uint32))
    assert np.array_equal(p.view(np.uint32), tp.view(np.uint32))


def test_lars_first_step_closed_form():
    h = dict(LARS, weight_decay=0.0)
    n = 4096
    p0 = synth.params(n, seed=6).numpy()
    p = p0.copy()
    oracle.optim32bit_layerwise_step("lars", p, synth.grads(n, step=1).numpy(), np.zeros(n, np.float32), None,
                                     step=1, trust_coefficient=ETA, **h)
    # v = lr * eta |w| / |g| * g  ->  |w' - w| = lr * eta * |w|
    dn = np.linalg.norm(p.astype(np.float64) - p0)
    assert dn == pytest.approx(h["lr"] * ETA * np.linalg.norm(p0.astype(np.float64)), rel=1e-4)


def test_lars_zero_norm_falls_back_to_lr():
    n = 64
    a = oracle.optim32bit_layerwise_step("lars", np.zeros(n, np.float32), synth.grads(n, step=1).numpy(),
                                         np.zeros(n, np.float32), None, step=1, trust_coefficient=ETA, **LARS)
    assert a == np.float32(LARS["lr"])
    a = oracle.optim32bit_layerwise_step("lars", synth.params(n).numpy(), np.zeros(n, np.float32),
                                         np.zeros(n, np.float32), None, step=1, trust_coefficient=ETA, **LARS)
    assert a == np.float32(LARS["lr"])


@pytest.mark.parametrize("kind", ["lamb", "lars"])
def test_8bit_layerwise_is_32bit_plus_block_quantization(kind):
    h = dict(LAMB if kind == "lamb" else LARS)
    n, B = 4 * 2048 + 901, 2048
    Qs, Qu = oracle.dynamic_codebook(True), oracle.dynamic_codebook(False)
    p = synth.params(n).numpy()
    g = synth.grads(n, step=3).numpy()
    s1, a1 = (t.numpy() for t in synth.random_state(n, seed=1, scale=1e-3))
    s2, a2 = (t.numpy() for t in synth.random_state(n, seed=2, scale=1e-6))
    m32 = oracle.dequantize_blockwise(Qs, s1, a1, B)
    r32 = oracle.dequantize_blockwise(Qu, s2, a2, B)
    p32 = p.copy()
    a32 = oracle.optim32bit_layerwise_step(kind, p32, g, m32, r32 if kind == "lamb" else None, step=3,
                                           trust_coefficient=ETA, **h)
    ea1, es1 = oracle.quantize_blockwise(Qs, m32, B)
    p8, s1b, a1b, s2b, a2b = p.copy(), s1.copy(), a1.copy(), s2.copy(), a2.copy()
    a8 = oracle.optim8bit_layerwise_step(kind, p8, g, s1b, s2b if kind == "lamb" else None, a1b,
                                         a2b if kind == "lamb" else None, step=3, trust_coefficient=ETA, **h)
    assert a8 == a32
    assert np.array_equal(p8.view(np.uint32), p32.view(np.uint32))
    assert np.array_equal(s1b, es1) and np.array_equal(a1b.view(np.uint32), ea1.view(np.uint32))
    if kind == "lamb":
        ea2, es2 = oracle.quantize_blockwise(Qu, r32, B)
        assert np.array_equal(s2b, es2) and np.array_equal(a2b.view(np.uint32), ea2.view(np.uint32))


@pytest.mark.parametrize("kind", ["lamb", "lars"])
def test_8bit_layerwise_tracks_32bit(kind):
    h = dict(LAMB if kind == "lamb" else LARS)
    n = 1 << 18
    p0 = synth.params(n).numpy()
    p8, p32 = p0.copy(), p0.copy()
    s1, a1 = (t.numpy() for t in synth.zero_state(n))
    s2, a2 = (t.numpy() for t in synth.zero_state(n))
    m, r = np.zeros(n, np.float32), np.zeros(n, np.float32)
    for t in range(1, 11):
        g = synth.grads(n, step=t).numpy()
        oracle.optim8bit_layerwise_step(kind, p8, g, s1, s2, a1, a2, step=t, trust_coefficient=ETA, **h)
        oracle.optim32bit_layerwise_step(kind, p32, g, m, r, step=t, trust_coefficient=ETA, **h)
    u8, u32 = p8.astype(np.float64) - p0, p32.astype(np.float64) - p0
    agg = np.sum(np.abs(u8 - u32)) / np.sum(np.abs(u32))
    assert agg <= 0.05, agg


@pytest.mark.parametrize("kind", ["lamb", "lars"])
def test_forced_scale_teacher_forcing(kind):
    """Teacher forcing (reading L3): forcing the oracle's own scale reproduces the unforced step bit
    for bit; a forced scale of 0 freezes LAMB's parameters (w - 0*u = w) while the moments still
    advance exactly as in the unforced step, and reduces LARS to w - beta*v."""
    n = 5000
    hp = dict(synth.HPARAMS[kind])
    eta = hp.pop("trust_coefficient", 0.001)
    two = kind == "lamb"

    def state():
        p = synth.params(n, seed=3).numpy()
        s1, a1 = (t.numpy() for t in synth.random_state(n, seed=4, scale=1e-3))
        s2, a2 = (t.numpy() for t in synth.random_state(n, seed=5, scale=1e-6))
        return [p, s1, s2 if two else None, a1, a2 if two else None]

    g = synth.grads(n, step=2, seed=6).numpy()
    a, b = state(), state()
    sa = oracle.optim8bit_layerwise_step(kind, a[0], g, a[1], a[2], a[3], a[4], step=2, trust_coefficient=eta, **hp)
    sb = oracle.optim8bit_layerwise_step(kind, b[0], g, b[1], b[2], b[3], b[4], step=2, trust_coefficient=eta,
                                         forced_scale=sa, **hp)
    assert sb == sa
    for x, y in zip(a, b):
        if x is not None:
            assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
    c = state()
    p0 = c[0].copy()
    v0 = oracle.dequantize_blockwise(oracle.dynamic_codebook(True), c[1], c[3])
    oracle.optim8bit_layerwise_step(kind, c[0], g, c[1], c[2], c[3], c[4], step=2, trust_coefficient=eta,
                                    forced_scale=0.0, **hp)
    if kind == "lamb":
        assert np.array_equal(c[0], p0)
        assert np.array_equal(c[1], a[1]) and np.array_equal(c[2], a[2])
    else:
        v = (np.float32(hp["beta1"]) * v0).astype(np.float32)
        assert np.array_equal(c[0], (p0 - v).astype(np.float32))
