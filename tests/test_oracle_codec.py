"""Pins for the oracle's block-wise codec (Eq.4; dequantization P:71; G3, G5, G7).

Checks: worked examples, absmax = np.max(np.abs(block)),
codes = brute-force argmin of the IEEE fp32 quotient x/N computed by numpy,
dequantization = numpy fp32 Q[code]*N, the half-gap round-trip bound, block
independence, outlier isolation and determinism across thread counts."""
import numpy as np
import pytest

import oracle
import synth


def brute_codes(Q, x, B):
    x = np.asarray(x, np.float32)
    out = np.zeros(x.size, np.uint8)
    Q64 = Q.astype(np.float64)
    for s in range(0, x.size, B):
        blk = x[s:s + B]
        N = np.float32(np.max(np.abs(blk))) if blk.size else np.float32(0)
        y = (blk / N).astype(np.float32) if N > 0 else np.zeros_like(blk)  # IEEE fp32 division
        out[s:s + B] = np.argmin(np.abs(Q64[None, :] - y.astype(np.float64)[:, None]), axis=1)
    return out


@pytest.fixture(scope="module")
def Qs():
    return oracle.dynamic_codebook(True)


@pytest.fixture(scope="module")
def Qu():
    return oracle.dynamic_codebook(False)


def test_spec_block_example(Qs):
    # T = [1, 0.5, 0.25, 0.125], B = 2 -> absmax [1, 0.25], identical code patterns
    absmax, codes = oracle.quantize_blockwise(Qs, np.array([1.0, 0.5, 0.25, 0.125], np.float32), 2)
    assert absmax.tolist() == [1.0, 0.25]
    assert codes[0] == codes[2] and codes[1] == codes[3]
    assert codes[0] == 255  # +1.0


def test_block_shapes(Qs):
    # n = 5000, B = 2048 -> 3 blocks 2048 / 2048 / 904
    x = synth.params(5000, seed=3).numpy()
    absmax, codes = oracle.quantize_blockwise(Qs, x, 2048)
    assert absmax.size == 3 and codes.size == 5000
    for b, (s, e) in enumerate([(0, 2048), (2048, 4096), (4096, 5000)]):
        assert absmax[b] == np.max(np.abs(x[s:e]))


@pytest.mark.parametrize("n,B", [(1, 2048), (17, 2048), (2047, 2048), (2049, 2048), (20000, 2048), (999, 64),
                                 (100, 1)])
@pytest.mark.parametrize("signed", [True, False])
def test_codes_match_brute_force(Qs, Qu, n, B, signed):
    Q = Qs if signed else Qu
    x = synth.params(n, seed=n + B, std=1.0).numpy()
    if not signed:
        x = x * x
    absmax, codes = oracle.quantize_blockwise(Q, x, B)
    assert np.array_equal(codes, brute_codes(Q, x, B))
    deq = oracle.dequantize_blockwise(Q, codes, absmax, B)
    np_deq = (Q[codes] * np.repeat(absmax, B)[:n]).astype(np.float32)
    assert np.array_equal(deq.view(np.uint32), np_deq.view(np.uint32))


@pytest.mark.parametrize("signed", [True, False])
def test_half_gap_bound_and_absmax_exactness(Qs, Qu, signed):
    Q = Qs if signed else Qu
    rng = np.random.default_rng(5)
    x = rng.standard_normal(64 * 2048).astype(np.float32) * np.float32(1e-3)
    x[rng.integers(0, x.size, 40)] *= 100  # outliers
    if not signed:
        x = np.abs(x)
    absmax, codes = oracle.quantize_blockwise(Q, x, 2048)
    deq = oracle.dequantize_blockwise(Q, codes, absmax, 2048)
    # the worst case distance to the nearest code over the normalized range [-1, 1]
    # ([0, 1] unsigned): half the largest gap, or the distance from -1 to Q[0]
    Q64 = Q.astype(np.float64)
    half_gap = max(np.max(np.diff(Q64)) / 2, Q64[0] + 1.0 if signed else 0.0)
    N = np.repeat(absmax, 2048).astype(np.float64)
    err = np.abs(deq.astype(np.float64) - x.astype(np.float64))
    # + 2^-23 N covers the binary32 roundings of x/N and of Q[c]*N
    assert np.all(err <= (half_gap + 2.0 ** -23) * N)
    # G3: a positive block maximum round-trips exactly; a negative one maps to Q[0]*N
    for b in range(absmax.size):
        blk = x[b * 2048:(b + 1) * 2048]
        i = int(np.argmax(np.abs(blk)))
        if blk[i] > 0:
            assert deq[b * 2048 + i] == blk[i]
        else:
            assert codes[b * 2048 + i] == 0 and deq[b * 2048 + i] == Q[0] * absmax[b]


def test_outlier_isolation(Qs):
    # S:175 / P:112: an outlier in block 0 leaves block 1's codes and absmax bit-identical
    x = np.random.default_rng(0).standard_normal(4096).astype(np.float32)
    a0, c0 = oracle.quantize_blockwise(Qs, x, 2048)
    x2 = x.copy()
    x2[0] = 100.0
    a1, c1 = oracle.quantize_blockwise(Qs, x2, 2048)
    assert a0[1] == a1[1] and np.array_equal(c0[2048:], c1[2048:])
    assert a1[0] == 100.0


def test_zero_block(Qs, Qu):
    x = np.zeros(3000, np.float32)
    for Q, zero_code in ((Qs, 127), (Qu, 0)):
        absmax, codes = oracle.quantize_blockwise(Q, x, 2048)
        assert np.all(absmax == 0) and np.all(codes == zero_code)
        assert np.all(oracle.dequantize_blockwise(Q, codes, absmax, 2048) == 0)


def test_idempotence_positive_max_blocks(Qs):
    # quantize(dequantize(quantize(T))) == quantize(T) when each block's max is positive (G3)
    x = np.abs(np.random.default_rng(2).standard_normal(16 * 2048)).astype(np.float32)
    x *= np.sign(np.random.default_rng(3).standard_normal(x.size)).astype(np.float32)
    for b in range(16):
        blk = x[b * 2048:(b + 1) * 2048]
        i = np.argmax(np.abs(blk))
        blk[i] = abs(blk[i])
    a, c = oracle.quantize_blockwise(Qs, x, 2048)
    a2, c2 = oracle.quantize_blockwise(Qs, oracle.dequantize_blockwise(Qs, c, a, 2048), 2048)
    assert np.array_equal(c, c2) and np.array_equal(a, a2)


@pytest.mark.parametrize("signed", [True, False])
def test_linear_type_keeps_exact_zeros(signed):
    """Reading L0: a zero element of a block with a nonzero absmax decodes to exactly 0 through the
    linear type (with the rejected symmetric -1 + 2i/255 grid it would decode to +-N/255)."""
    Q = oracle.linear_codebook(signed)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(5000).astype(np.float32)
    if not signed:
        x = np.abs(x)
    x[::4] = 0.0
    absmax, codes = oracle.quantize_blockwise(Q, x)
    d = oracle.dequantize_blockwise(Q, codes, absmax)
    assert np.all(d[::4] == 0.0) and np.all(absmax > 0)
