"""Pins for the oracle's quantile functions (App F.2 Eq.5, App G SRAM-Quantiles
P:432-444; readings Q1-Q5 in DESIGN.md section 3).  Each check is fixed by something other than
the oracle itself: closed-form order statistics, numpy's sort, the normal quantile function, exact
rational means, symmetry."""
from fractions import Fraction

import numpy as np
import pytest
from scipy.stats import norm

import oracle

J = np.arange(257)


@pytest.mark.parametrize("m", [1, 2, 7, 256, 257, 1000, 4095, 4096, 5000])
def test_exact_quantiles_of_a_permuted_range(m):
    # the j-th quantile of {0..m-1} is the value at sorted index floor(j*m/257) = that index (Q2)
    x = np.random.default_rng(m).permutation(m).astype(np.float32)
    want = np.array([(j * m) // 257 for j in range(257)], np.float32)
    np.testing.assert_array_equal(oracle.exact_quantiles(x), want)


@pytest.mark.parametrize("n", [1, 33, 4096, 100_003])
def test_exact_quantiles_match_numpy_sort(n):
    x = np.random.default_rng(n).standard_normal(n).astype(np.float32)
    want = np.sort(x)[(J * n) // 257]
    np.testing.assert_array_equal(oracle.exact_quantiles(x), want)


@pytest.mark.parametrize("n", [5, 4096, 10_000])
def test_sram_single_chunk_is_exact(n):
    x = np.random.default_rng(7).standard_normal(n).astype(np.float32)
    np.testing.assert_array_equal(oracle.sram_quantiles(x, subset=max(n, 4096)), oracle.exact_quantiles(x))


def test_sram_constant_chunks_average_exactly():
    # chunk c holds the constant v_c, so all its quantiles are v_c and the estimate is mean(v) (Q4);
    # the last chunk is short (Q3) and still weighs 1
    rng = np.random.default_rng(3)
    vals = rng.integers(-1000, 1000, size=9).astype(np.float32) / 8
    S = 4096
    x = np.concatenate([np.full(S if c < 8 else 123, v, np.float32) for c, v in enumerate(vals)])
    mean = sum(Fraction(float(v)) for v in vals) / len(vals)
    want = np.float32(float(mean))  # sum of multiples of 1/8 is exact in double; one rounding
    np.testing.assert_array_equal(oracle.sram_quantiles(x, S), np.full(257, want, np.float32))


def test_sram_two_ranges_closed_form():
    # chunk 0 = a permutation of 0..4095, chunk 1 = 4096..8191: mean of the j-th quantiles is
    # floor(j*4096/257) + 2048
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.permutation(4096), 4096 + rng.permutation(4096)]).astype(np.float32)
    want = np.array([(j * 4096) // 257 + 2048 for j in range(257)], np.float32)
    np.testing.assert_array_equal(oracle.sram_quantiles(x, 4096), want)


def test_sram_permutation_invariant_within_chunks():
    rng = np.random.default_rng(2)
    x = rng.standard_normal(4096 * 5 + 77).astype(np.float32)
    y = x.copy()
    for c in range(0, y.size, 4096):
        y[c:c + 4096] = rng.permutation(y[c:c + 4096])
    np.testing.assert_array_equal(oracle.sram_quantiles(x), oracle.sram_quantiles(y))


def test_sram_estimates_the_normal_quantile_function():
    # "samples quantiles estimated via eCDFs are asymptotically unbiased estimators of the
    # population quantile": 512 chunks of N(0,1) land near Phi^-1(j/257)
    x = np.random.default_rng(5).standard_normal(4096 * 512).astype(np.float32)
    q = oracle.sram_quantiles(x)
    p = norm.ppf(J / 257)
    assert np.abs(q[1:256] - p[1:256]).max() < 0.03
    assert np.abs(q[16:241] - p[16:241]).max() < 0.01
    assert np.all(np.diff(q) >= 0)


def test_quantile_codebook_uniform_closed_form():
    # quantiles of U(-1,1) at j/256 spacing: Q_j = -1 + j/128 -> Eq.5 midpoints -1 + (2i+1)/256,
    # largest magnitude 255/256 -> code_i = (2i - 255)/255 (Q5)
    Q = (-1.0 + J / 128.0).astype(np.float32)
    want = (np.float64(2 * np.arange(256) - 255) / 255.0).astype(np.float32)
    np.testing.assert_array_equal(oracle.quantile_codebook(Q), want)


def test_quantile_codebook_symmetry_and_range():
    rng = np.random.default_rng(9)
    half = np.sort(rng.standard_normal(128).astype(np.float32))
    half = half - half[-1] - np.float32(0.5)  # all negative, ascending
    Q = np.concatenate([half, [np.float32(0.0)], -half[::-1]]).astype(np.float32)
    assert Q.size == 257 and np.all(np.diff(Q) > 0)
    c = oracle.quantile_codebook(Q)
    np.testing.assert_array_equal(c[::-1], -c)          # antisymmetric quantiles -> antisymmetric table
    assert np.abs(c).max() == np.float32(1.0)
    assert np.all(np.diff(c) > 0)
    # Eq.5 by hand for one entry
    i = 17
    m = (np.float64(Q[i]) + np.float64(Q[i + 1])) / 2
    M = max(abs((np.float64(Q[k]) + np.float64(Q[k + 1])) / 2) for k in range(256))
    assert c[i] == np.float32(m / M)


def test_quantile_codebook_rejects_all_zero():
    with pytest.raises(ValueError):
        oracle.quantile_codebook(np.zeros(257, np.float32))
