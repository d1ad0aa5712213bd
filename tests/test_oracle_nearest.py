"""Pins for the oracle's nearest-code search (Eq.3; tie rule G6).

The oracle uses a binary search plus a two-neighbour compare.  Here it is checked
against brute force: np.argmin over all 256 exact float64 distances (np.argmin
returns the FIRST minimum, i.e. ties go to the lower index)."""
import numpy as np
import pytest

import oracle


def brute(Q, y):
    Q64 = Q.astype(np.float64)
    y64 = np.asarray(y, dtype=np.float32).astype(np.float64)
    return np.argmin(np.abs(Q64[None, :] - y64[:, None]), axis=1).astype(np.uint8)


def adversarial_inputs(Q):
    Q64 = Q.astype(np.float64)
    mids = (Q64[:-1] + Q64[1:]) / 2  # exact in float64
    pts = []
    for base in (np.float32(mids), Q):
        b = np.asarray(base, dtype=np.float32)
        pts.append(b)
        up, dn = b.copy(), b.copy()
        for _ in range(4):
            up = np.nextafter(up, np.float32(np.inf))
            dn = np.nextafter(dn, np.float32(-np.inf))
            pts += [up.copy(), dn.copy()]
    # the fp32 values bracketing every midpoint from below and above
    lo = np.float32(mids)
    lo = np.where(lo.astype(np.float64) > mids, np.nextafter(lo, np.float32(-np.inf)), lo)
    hi = np.nextafter(lo, np.float32(np.inf))
    pts += [lo, hi]
    pts.append(np.array([0.0, -0.0, 1.0, -1.0, 1e-30, -1e-30, 1e-45, 2.0, -2.0], np.float32))
    return np.concatenate(pts).astype(np.float32)


@pytest.mark.parametrize("signed", [True, False])
def test_adversarial_matches_brute_force(signed):
    Q = oracle.dynamic_codebook(signed)
    y = adversarial_inputs(Q)
    assert np.array_equal(oracle.nearest_code(Q, y), brute(Q, y))


@pytest.mark.parametrize("signed", [True, False])
def test_exact_ties_go_to_lower_index(signed):
    Q = oracle.dynamic_codebook(signed)
    Q64 = Q.astype(np.float64)
    mids = (Q64[:-1] + Q64[1:]) / 2
    exact = np.float32(mids).astype(np.float64) == mids
    assert exact.sum() > 50  # ties are real for this table (G6)
    k = np.nonzero(exact)[0]
    got = oracle.nearest_code(Q, np.float32(mids[k]))
    assert np.array_equal(got, k.astype(np.uint8))


@pytest.mark.parametrize("signed", [True, False])
def test_random_matches_brute_force(signed):
    rng = np.random.default_rng(11)
    Q = oracle.dynamic_codebook(signed)
    lo = -1.0 if signed else 0.0
    y = np.concatenate([
        rng.uniform(lo, 1.0, 20000),
        np.sign(rng.uniform(lo, 1.0, 20000)) * 10.0 ** rng.uniform(-9, 0, 20000),
    ]).astype(np.float32)
    assert np.array_equal(oracle.nearest_code(Q, y), brute(Q, y))
