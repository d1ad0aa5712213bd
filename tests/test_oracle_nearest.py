"""Pins for the oracle's nearest-code search (Eq.3; tie rule G6).

The oracle uses a binary search plus a two-neighbour compare.  Here it is checked
against brute force: np.argmin over all 256 float64 distances (np.argmin returns the
FIRST minimum, i.e. ties go to the lower index) -- exact for the dynamic tables, whose
midpoints are never far below the codes around them -- and, for any table, against
an exact brute force over rational distances (fractions.Fraction)."""
from fractions import Fraction

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


def brute_exact(Q, y):
    """argmin_j |Q_j - y| over exact rationals, first minimum (ties -> lower index, G6)."""
    Qf = [Fraction(float(q)) for q in Q]
    out = []
    for v in np.asarray(y, np.float32):
        yv = Fraction(float(v))
        d = [abs(q - yv) for q in Qf]
        out.append(d.index(min(d)))
    return np.array(out, np.uint8)


def _exact_tables():
    sym = (np.arange(256, dtype=np.float64) * 2 / 255 - 1).astype(np.float32)   # no 0: a midpoint AT 0
    wide = np.sort(np.concatenate([-np.logspace(-30, 0, 128), np.logspace(-30, 0, 128)])).astype(np.float32)
    return {"dynamic_signed": oracle.dynamic_codebook(True), "symmetric_no_zero": sym, "wide_range": wide}


@pytest.mark.parametrize("name", ["dynamic_signed", "symmetric_no_zero", "wide_range"])
def test_matches_exact_rational_brute_force(name):
    """Tiny inputs next to a midpoint at (or near) 0 are where a binary64 subtraction y - Q loses y (y = 1e-45,
    Q = 1/255): the oracle must still return the exactly nearest code (Eq.3; G6)."""
    Q = _exact_tables()[name]
    rng = np.random.default_rng(5)
    tiny = np.array([1e-45, 3e-45, 1e-40, 1e-38, 1e-30, 1e-20, 4.3e-19, 1e-10], np.float32)
    mids = ((Q[:-1].astype(np.float64) + Q[1:]) / 2).astype(np.float32)
    y = np.concatenate([tiny, -tiny, [0.0, -0.0, 1.0, -1.0], mids, np.nextafter(mids, np.float32(1)),
                        np.nextafter(mids, np.float32(-1)), rng.uniform(-1, 1, 300),
                        np.sign(rng.uniform(-1, 1, 300)) * 10.0 ** rng.uniform(-40, 0, 300)]).astype(np.float32)
    assert np.array_equal(oracle.nearest_code(Q, y), brute_exact(Q, y))


def test_exact_compare_fixes_lost_subtraction():
    """The case that motivated the exact compare: y = 1e-45 is strictly closer to +1/255 than to -1/255,
    but the binary64 distances both round to 1/255 (a false tie -> the lower index)."""
    Q = _exact_tables()["symmetric_no_zero"]
    assert int(oracle.nearest_code(Q, np.float32(1e-45))[0]) == 128
    assert int(oracle.nearest_code(Q, np.float32(-1e-45))[0]) == 127
    assert int(oracle.nearest_code(Q, np.float32(0.0))[0]) == 127       # exact tie -> lower
