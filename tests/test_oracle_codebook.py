"""Pins for the oracle's dynamic data type (P:90 S2.3, P:118 S3.2; readings G1, G2, G4).

Nothing here re-calls the oracle's own formula: the tables are checked against an exact
rational enumeration done with Python Fractions, against structural invariants the
paper states, and against golden values/hashes from an independent enumeration
(tests/golden/codebook_appB.txt)."""
import hashlib
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "codebook_appB.txt")


def rn_f32(q: Fraction) -> np.float32:
    """Correctly rounded (nearest, ties-to-even) binary32 value of an exact rational."""
    c = np.float32(float(q))  # within one ulp of the answer
    cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
    best = min(cands, key=lambda v: (abs(Fraction(float(v)) - q), int(np.float32(v).view(np.uint32)) & 1))
    return np.float32(best)


def exact_values(signed: bool):
    """Enumerate the G1 reading in exact arithmetic: for z = 0..6 zero bits and F fraction
    bits (F = 6 - z signed, 7 - z unsigned), magnitude 10^-z * (0.1 + 0.9 (f + 1/2) / 2^F)
    = (2L + 18f + 9) / (20 L 10^z) with L = 2^F; plus the two special values 0 and +1."""
    vals = [Fraction(0), Fraction(1)]
    for z in range(7):
        F = (6 - z) if signed else (7 - z)
        L = 2 ** F
        for f in range(L):
            mag = Fraction(2 * L + 18 * f + 9, 20 * L * 10 ** z)
            vals.append(mag)
            if signed:
                vals.append(-mag)
    return vals


@pytest.mark.parametrize("signed", [True, False])
def test_matches_exact_rational_enumeration(signed):
    Q = oracle.dynamic_codebook(signed)
    ex = exact_values(signed)
    assert len(ex) == 256
    expected = np.sort(np.array([rn_f32(v) for v in ex], dtype=np.float32))
    assert np.array_equal(Q.view(np.uint32), expected.view(np.uint32))


@pytest.mark.parametrize("signed", [True, False])
def test_invariants(signed):
    Q = oracle.dynamic_codebook(signed)
    assert Q.dtype == np.float32 and Q.shape == (256,)
    assert np.all(np.diff(Q.astype(np.float64)) > 0), "strictly ascending, 256 distinct"
    assert Q[-1] == np.float32(1.0), "max = +1 (range [-1, 1], P:90)"
    zero_idx = 127 if signed else 0
    assert Q[zero_idx] == 0.0
    if signed:
        assert Q[0] < 0 and Q[0] > -1.0  # G3: -1 is not representable under G1
    else:
        assert Q.min() == 0.0
    pos = Q[(Q > 0) & (Q < 1)].astype(np.float64)
    # decade tiling: decade z holds 2^(6-z) (signed) / 2^(7-z) (unsigned) magnitudes in (0.1*10^-z, 10^-z)
    for z in range(7):
        hi, lo = 10.0 ** (-z), 10.0 ** (-z - 1)
        cnt = int(np.sum((pos > lo) & (pos < hi)))
        assert cnt == (2 ** (6 - z) if signed else 2 ** (7 - z)), (z, cnt)
    # ~7 decades of range: smallest nonzero magnitude between 1e-7 and 1e-6
    assert 1e-7 < pos.min() < 1e-6
    if signed:
        neg = -Q[Q < 0].astype(np.float64)
        assert np.array_equal(np.sort(neg), pos), "signed table is symmetric apart from +1"
        # "precision as high as 1/63": the top decade has >= 63 levels
        assert np.sum(pos > 0.1) >= 63


def _golden():
    vals, hashes = {}, {}
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        table, key, val = line.split()
        if key == "sha256_prefix":
            hashes[table] = val
        else:
            vals[(table, int(key))] = np.float32(float(val))
    return vals, hashes


def test_golden_appendix_b():
    vals, hashes = _golden()
    tabs = {"signed": oracle.dynamic_codebook(True), "unsigned": oracle.dynamic_codebook(False)}
    for (table, idx), v in vals.items():
        assert tabs[table][idx] == v, (table, idx, tabs[table][idx], v)
    for table, pre in hashes.items():
        h = hashlib.sha256(tabs[table].astype("<f4").tobytes()).hexdigest()
        assert h.startswith(pre), (table, h)


@pytest.mark.parametrize("signed", [True, False])
def test_every_code_round_trips(signed):
    """quantize(dequantize(i)) = i for every code (BASELINE north_star invariant)."""
    Q = oracle.dynamic_codebook(signed)
    assert np.array_equal(oracle.nearest_code(Q, Q), np.arange(256, dtype=np.uint8))


@pytest.mark.parametrize("signed", [True, False])
def test_linear_codebook(signed):
    """Linear type (T3 caption; reading L0): 256 evenly spaced values, max +1, an exact 0
    (zero-initialized states must round-trip, Eq.2), the signed type symmetric apart from +1."""
    Q = oracle.linear_codebook(signed).astype(np.float64)
    assert Q.size == 256 and np.all(np.diff(Q) > 0)
    assert Q[-1] == 1.0 and Q[0] == (-127 / 128 if signed else 0.0)
    step = (Q[-1] - Q[0]) / 255
    assert np.max(np.abs(np.diff(Q) - step)) <= 2 * np.spacing(np.float32(1.0))   # even spacing
    assert Q[127 if signed else 0] == 0.0                                            # exact zero
    if signed:
        assert np.array_equal(Q[:255], -Q[:255][::-1])                              # symmetric but +1
        assert step == 1 / 128
    assert np.array_equal(oracle.nearest_code(oracle.linear_codebook(signed), oracle.linear_codebook(signed)),
                          np.arange(256, dtype=np.uint8))
