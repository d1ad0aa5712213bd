"""Pins for the oracle's optimizer steps (Eq.1, Eq.2 P:52-60, S3 P:96-98; G8-G14).

* hand arithmetic and the t = 1 closed form of bias-corrected Adam;
* the 32-bit step against torch.optim.{Adam, AdamW, SGD} on CPU in fp32 (library
  routines; torch rounds a mathematically equal expression differently, so rtol 1e-5);
* the 8-bit step equals dequantize -> 32-bit step -> explicit block quantization,
  bit-for-bit (SPEC S:345 / acceptance 9), with the codec pinned in test_oracle_codec;
* 8-bit vs 32-bit Adam over 10 steps within quantization error;
* results independent of the oracle's thread count (block independence)."""
import numpy as np
import pytest
import torch

import oracle
import synth


def test_adam_hand_arithmetic_no_bias_correction():
    # m=r=0, g=0.1 -> m'=0.01, r'=1e-5, dw ~= -0.0031623
    p = np.array([0.5], np.float32)
    m = np.zeros(1, np.float32)
    r = np.zeros(1, np.float32)
    oracle.optim32bit_step("adam", p, np.array([0.1], np.float32), m, r, lr=1e-3, beta1=0.9, beta2=0.999,
                           eps=1e-8, bias_correction=False, step=1)
    assert m[0] == pytest.approx(0.01, rel=1e-6)
    assert r[0] == pytest.approx(1e-5, rel=1e-5)
    assert p[0] - 0.5 == pytest.approx(-0.0031623, rel=1e-4)


def test_momentum_hand_arithmetic():
    # m=1, g=1, beta=0.9, lr=0.1 -> m'=1.9, w decreases by 0.19
    p = np.array([1.0], np.float32)
    m = np.array([1.0], np.float32)
    oracle.optim32bit_step("momentum", p, np.array([1.0], np.float32), m, None, lr=0.1, beta1=0.9,
                           bias_correction=False, step=2)
    assert m[0] == np.float32(1.9)
    assert p[0] == pytest.approx(1.0 - 0.19, rel=1e-6)
    # Eq.1 initialization m_0 = g_0 follows from the zero state
    m0 = np.zeros(3, np.float32)
    g0 = np.array([2.0, -1.0, 0.25], np.float32)
    oracle.optim32bit_step("momentum", np.zeros(3, np.float32), g0, m0, None, lr=0.1, beta1=0.9, step=1)
    assert np.array_equal(m0, g0)


@pytest.mark.parametrize("hp", ["adam", "adam_paper"])
def test_bias_corrected_first_step_closed_form(hp):
    # t = 1 from zero state: m = (1-b1) g, r = (1-b2) g^2, bias correction -> dp = -lr g/(|g| + eps)
    h = dict(synth.HPARAMS[hp])
    g = synth.grads(1 << 16, step=1).numpy()
    p0 = synth.params(1 << 16).numpy()
    p = p0.copy()
    oracle.optim32bit_step("adam", p, g, np.zeros_like(p), np.zeros_like(p), step=1, **h)
    dp = p.astype(np.float64) - p0
    expect = -h["lr"] * g.astype(np.float64) / (np.abs(g.astype(np.float64)) + h["eps"])
    # rtol 1e-6: the fp32 ops of the step contribute a few 1e-7 relative to dp; the final
    # rounding of w is at most half an ulp of |w| (atol)
    np.testing.assert_allclose(dp, expect, rtol=1e-6, atol=np.spacing(np.abs(p0).astype(np.float32)).max())


def _torch_run(kind, h, p0, gs):
    w = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    if kind == "momentum":
        opt = torch.optim.SGD([w], lr=h["lr"], momentum=h["beta1"], dampening=0, weight_decay=h["weight_decay"])
    elif kind == "adamw":
        opt = torch.optim.AdamW([w], lr=h["lr"], betas=(h["beta1"], h["beta2"]), eps=h["eps"],
                                weight_decay=h["weight_decay"], foreach=False)
    else:
        opt = torch.optim.Adam([w], lr=h["lr"], betas=(h["beta1"], h["beta2"]), eps=h["eps"],
                               weight_decay=h["weight_decay"], foreach=False)
    for g in gs:
        w.grad = torch.from_numpy(g.copy())
        opt.step()
    st = opt.state[w]
    m = st["momentum_buffer" if kind == "momentum" else "exp_avg"].numpy()
    r = None if kind == "momentum" else st["exp_avg_sq"].numpy()
    return w.detach().numpy(), m, r


@pytest.mark.parametrize("kind,hp,wd", [("adam", "adam", 0.0), ("adam", "adam", 0.01), ("adam", "adam_paper", 0.0),
                                        ("adamw", "adamw", 0.01), ("momentum", "momentum", 0.0),
                                        ("momentum", "momentum", 1e-4)])
def test_32bit_step_matches_torch_optim(kind, hp, wd):
    h = dict(synth.HPARAMS[hp])
    h["weight_decay"] = wd
    if kind == "momentum":
        h["bias_correction"] = False
    n = 4096
    p0 = synth.params(n).numpy()
    gs = [synth.grads(n, step=t).numpy() for t in range(1, 6)]
    p, m, r = p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    for t, g in enumerate(gs, start=1):
        oracle.optim32bit_step(kind, p, g, m, r, step=t, **h)
    tp, tm, tr = _torch_run(kind, h, p0, gs)
    # p accumulates lr-sized updates whose rounding differs by a few ulps of p
    np.testing.assert_allclose(p, tp, rtol=1e-6, atol=8 * np.spacing(np.abs(tp).max()))
    # m is a signed running sum: cancellation makes elementwise relative error meaningless
    # near m = 0, so the absolute bound is scaled by the state's magnitude.
    np.testing.assert_allclose(m, tm, rtol=1e-5, atol=1e-6 * np.abs(tm).max())
    if tr is not None:
        np.testing.assert_allclose(r, tr, rtol=1e-5, atol=1e-6 * np.abs(tr).max())


@pytest.mark.parametrize("kind", ["adam", "adamw", "momentum"])
def test_8bit_step_is_32bit_step_plus_block_quantization(kind):
    """dequantize -> 32-bit update -> requantize (Eq.4), p from fp32 states (G12)."""
    h = dict(synth.HPARAMS[kind])
    n, B = 5 * 2048 + 333, 2048
    Qs, Qu = oracle.dynamic_codebook(True), oracle.dynamic_codebook(False)
    p = synth.params(n).numpy()
    g = synth.grads(n, step=3).numpy()
    s1, a1 = (t.numpy() for t in synth.random_state(n, seed=1, scale=1e-3))
    s2, a2 = (t.numpy() for t in synth.random_state(n, seed=2, scale=1e-6))
    # reference composition
    m32 = oracle.dequantize_blockwise(Qs, s1, a1, B)
    r32 = oracle.dequantize_blockwise(Qu, s2, a2, B)
    p32 = p.copy()
    oracle.optim32bit_step(kind, p32, g, m32, r32, step=3, **h)
    ea1, es1 = oracle.quantize_blockwise(Qs, m32, B)
    # the 8-bit step
    p8, s1b, a1b, s2b, a2b = p.copy(), s1.copy(), a1.copy(), s2.copy(), a2.copy()
    oracle.optim8bit_step(kind, p8, g, s1b, s2b, a1b, a2b, step=3, **h)
    assert np.array_equal(p8.view(np.uint32), p32.view(np.uint32))
    assert np.array_equal(s1b, es1) and np.array_equal(a1b.view(np.uint32), ea1.view(np.uint32))
    if kind != "momentum":
        ea2, es2 = oracle.quantize_blockwise(Qu, r32, B)
        assert np.array_equal(s2b, es2) and np.array_equal(a2b.view(np.uint32), ea2.view(np.uint32))
    else:
        assert np.array_equal(s2b, s2)


def test_thread_count_independence():
    n = 37 * 2048 + 5
    h = synth.HPARAMS["adamw"]
    g = synth.grads(n, step=1).numpy()
    outs = []
    for nt in (1, 2, 8):
        p = synth.params(n).numpy()
        s1, a1 = (t.numpy() for t in synth.random_state(n, seed=4))
        s2, a2 = (t.numpy() for t in synth.random_state(n, seed=5, scale=1e-6))
        oracle.optim8bit_step("adamw", p, g, s1, s2, a1, a2, step=7, nthreads=nt, **h)
        outs.append((p, s1, s2, a1, a2))
    for o in outs[1:]:
        for x, y in zip(outs[0], o):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("kind", ["adam", "momentum"])
def test_8bit_tracks_32bit_within_quantization_error(kind):
    """SURVEY 8(c) P6 bounds, 10 steps on config 1 (1M elements, no outliers)."""
    h = synth.HPARAMS[kind]
    n = 1 << 20
    p0 = synth.params(n).numpy()
    p8, p32 = p0.copy(), p0.copy()
    s1, a1 = (t.numpy() for t in synth.zero_state(n))
    s2, a2 = (t.numpy() for t in synth.zero_state(n))
    m, r = np.zeros(n, np.float32), np.zeros(n, np.float32)
    for t in range(1, 11):
        g = synth.grads(n, step=t).numpy()
        oracle.optim8bit_step(kind, p8, g, s1, s2, a1, a2, step=t, nthreads=8, **h)
        oracle.optim32bit_step(kind, p32, g, m, r, step=t, **h)
    u8 = (p8.astype(np.float64) - p0)
    u32 = (p32.astype(np.float64) - p0)
    lr = h["lr"]
    agg = np.sum(np.abs(u8 - u32)) / np.sum(np.abs(u32))
    dp = np.abs(p8.astype(np.float64) - p32)
    assert agg <= 0.05, agg
    assert np.mean(dp) <= 0.1 * lr
    assert np.max(dp) <= 10 * lr
    if kind == "adam":
        rel = np.abs(u8 - u32) / np.maximum(np.abs(u32), 1e-30)
        assert np.median(rel) <= 0.05
