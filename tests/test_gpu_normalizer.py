"""GPU sweep of the normalization y = RN(x / N_b) (Eq.4, reading G7) as the kernels compute
it: a per-block reciprocal RN(1/N) and one Markstein correction per element, which
must equal IEEE binary32 division wherever the code depends on it.

Every block holds one N (its element 0, so absmax = N) and 2047 values x placed on each of the 255
decision boundaries of the table scaled by N, at -4..+3 ulps around RN(b_k * N), plus +-N and 0.
The N values are ALL 2^23 mantissas of the binade [1, 2), sampled mantissas of binades from the
bottom (2^-70) to the top (2^125) of the fast range, and N outside it (the block-uniform IEEE
fallback).  The kernel is q8_quantize_blockwise_dynamic (the step kernel's normalization and
search code).

Expected codes: the oracle's nearest-code step function (decision boundaries b_k found by bisection
over oracle.nearest_code, tests/test_gpu_parity.py) at y = RN32(x / N) computed in binary64 and
rounded once to binary32 -- double rounding is innocuous for a quotient of binary32 operands
(53 >= 2*24 + 2), so that is the correctly rounded binary32 quotient.  A sample of the blocks is
also compared with oracle.quantize_blockwise directly."""
import numpy as np
import pytest
import torch

import oracle
from test_gpu_parity import _boundaries, assert_same

pytestmark = pytest.mark.gpu
DEV = "cuda"
OFFS = range(-4, 4)            # ulps around RN(b_k * N)


@pytest.fixture(scope="module")
def q8():
    import paper_2110_02861_b200 as m
    return m


def _blocks(N, bnd_f32):
    """[nb, 2048] fp32 blocks: x[:, 0] = N, then every (boundary k, ulp offset d) pair, then
    -N (signed tables only; +N otherwise), +N, 0 and padding zeros."""
    nb = N.numel()
    k = torch.arange(255, device=DEV).repeat(len(OFFS))                      # 2040 slots
    d = torch.tensor(list(OFFS), device=DEV, dtype=torch.int32).repeat_interleave(255)
    x = torch.zeros(nb, 2048, dtype=torch.float32, device=DEV)
    x[:, 0] = N
    base = bnd_f32[k][None, :] * N[:, None]                                 # RN(b_k * N)
    # step by d ulps in the direction of increasing value, through the monotone integer key of the fp32
    # order (key = bits for x >= +0, -(|bits| + 1) for x <= -0), so steps may cross zero (boundaries at
    # the smallest denormals: a caller table whose midpoint is 0)
    bits = base.view(torch.int32)
    key = torch.where(bits >= 0, bits, -(bits & 0x7FFFFFFF) - 1) + d[None, :]
    sign = torch.tensor(-0x80000000, dtype=torch.int32, device=DEV)
    x[:, 1:2041] = torch.where(key >= 0, key, (-(key + 1)) | sign).view(torch.float32)
    x[:, 2041] = -N
    x[:, 2042] = N
    return x


def _expected(x, N, bnd64):
    y = (x.to(torch.float64) / N.to(torch.float64)[:, None]).to(torch.float32).to(torch.float64)
    return torch.searchsorted(bnd64, y.reshape(-1), right=True).reshape(x.shape)


def _sweep(q8, signed, N, chunk=1 << 17, Q=None):
    """Q None: the built-in dynamic table (q8_quantize_blockwise_dynamic); else the caller table Q through
    q8_quantize_blockwise (its own thresholds; the packed Markstein normalization when no threshold lies
    within 2^-39 of 0, else the IEEE division)."""
    generic = Q is not None
    if Q is None:
        Q = oracle.dynamic_codebook(signed)
    code_dev = torch.from_numpy(np.ascontiguousarray(Q, np.float32)).to(DEV)
    bnd = _boundaries(Q)
    bnd64 = torch.from_numpy(bnd).to(DEV)
    bnd32 = torch.from_numpy(bnd.astype(np.float32)).to(DEV)
    bad = 0
    for s in range(0, N.numel(), chunk):
        Nc = N[s:s + chunk]
        x = _blocks(Nc, bnd32)
        if not signed:
            x = x.abs()    # unsigned table: non-negative states; boundaries are all >= 0
        if generic:
            a, c = q8.quantize_blockwise(code_dev, x.reshape(-1))
        else:
            a, c = q8.quantize_blockwise_dynamic(signed, x.reshape(-1))
        assert torch.equal(a.view(torch.int32), Nc.abs().view(torch.int32)), "absmax != N"
        exp = _expected(x, Nc, bnd64)
        bad += int((c.view(x.shape).to(torch.int64) != exp).sum())
        del x, a, c, exp
    return bad


@pytest.mark.slow
@pytest.mark.parametrize("signed", [True, False])
def test_normalizer_all_mantissas(q8, signed):
    """All 2^23 mantissas of N in [1, 2) x 255 boundaries x 8 ulp offsets (1.7e10 elements)."""
    N = (torch.arange(1 << 23, dtype=torch.int32, device=DEV) + 0x3F800000).view(torch.float32)
    assert _sweep(q8, signed, N) == 0


@pytest.mark.parametrize("signed", [True, False])
def test_normalizer_binades(q8, signed):
    """Sampled mantissas (2^14 per binade) across the fast range 2^-70 <= N < 2^126, at its edges,
    and outside it (N < 2^-70 and N >= 2^126 take the IEEE-division fallback)."""
    g = torch.Generator(device=DEV)
    g.manual_seed(123)
    Ns = []
    for e in (-80, -71, -70, -69, -40, -20, -1, 0, 1, 20, 60, 100, 124, 125, 126, 127):
        m = torch.randint(0, 1 << 23, (1 << 14,), generator=g, device=DEV, dtype=torch.int32)
        m[:2] = torch.tensor([0, (1 << 23) - 1], device=DEV, dtype=torch.int32)   # binade ends
        Ns.append(((e + 127) << 23 | m).view(torch.float32))
    N = torch.cat(Ns)
    assert _sweep(q8, signed, N) == 0


@pytest.mark.parametrize("signed", [True, False])
def test_normalizer_blocks_vs_oracle_codec(q8, signed):
    """The same adversarial blocks for 256 N values (random mantissas in [1, 2) and two far binades)
    straight through oracle.quantize_blockwise: codes and absmax bit-exact."""
    g = torch.Generator(device=DEV)
    g.manual_seed(7)
    m = torch.randint(0, 1 << 23, (256,), generator=g, device=DEV, dtype=torch.int32)
    e = torch.tensor([127] * 128 + [127 - 60] * 64 + [127 + 100] * 64, device=DEV, dtype=torch.int32)
    N = (e << 23 | m).view(torch.float32)
    Q = oracle.dynamic_codebook(signed)
    x = _blocks(N, torch.from_numpy(_boundaries(Q).astype(np.float32)).to(DEV))
    if not signed:
        x = x.abs()
    x = x.reshape(-1)
    a, c = q8.quantize_blockwise_dynamic(signed, x)
    a_r, c_r = oracle.quantize_blockwise(Q, x.cpu().numpy())
    assert_same(a, a_r, "absmax")
    assert_same(c, c_r, "codes")


def _caller_tables():
    rng = np.random.default_rng(3)
    quant = oracle.quantile_codebook(oracle.exact_quantiles(rng.standard_normal(1 << 16).astype(np.float32)))
    tiny = oracle.dynamic_codebook(True).copy()
    assert tiny[127] == 0.0
    tiny[128], tiny[129] = np.float32(1e-13), np.float32(2e-13)
    return {
        "dynamic_signed": (True, oracle.dynamic_codebook(True)),
        "dynamic_unsigned": (False, oracle.dynamic_codebook(False)),
        "linear_signed": (True, oracle.linear_codebook(True)),      # exact 0 code: thresholds +-1/256
        "quantile": (True, quant),                                   # Eq.5 quantile data type
        # symmetric grid without 0: a threshold at exactly 0 -> the kernel keeps the IEEE division
        "symmetric_no_zero": (True, (np.arange(256, dtype=np.float64) * 2 / 255 - 1).astype(np.float32)),
        # codes 1e-13, 2e-13 next to 0: thresholds below 2^-39 -> the IEEE division
        "tiny_codes": (True, tiny),
        # 128 codes packed into [0.87, 1]: buckets of the top binade span up to ~9 codes -> the long launch
        # rejects the bucket table and keeps the 8-step descent
        "dense_top": (True, np.concatenate([np.linspace(-1, 0.86, 128), np.linspace(0.87, 1, 128)]).astype(np.float32)),
    }


@pytest.mark.parametrize("name", ["dynamic_signed", "dynamic_unsigned", "linear_signed", "quantile",
                                  "symmetric_no_zero", "tiny_codes", "dense_top"])
def test_normalizer_binades_caller_table(q8, name):
    """The generic (caller-table) quantizer on the adversarial blocks: sampled mantissas (2^12 per binade)
    across and outside the fast range, every decision boundary of the table at -4..+3 ulps.  The launches
    are long enough (>= 16 blocks per CTA) for the per-CTA bucket table (q8_quant_kernel.cuh), so this
    covers it, its rejection (dense_top) and both normalizations."""
    signed, Q = _caller_tables()[name]
    g = torch.Generator(device=DEV)
    g.manual_seed(321)
    Ns = []
    for e in (-80, -70, -69, -40, -1, 0, 1, 60, 125, 126):
        m = torch.randint(0, 1 << 23, (1 << 12,), generator=g, device=DEV, dtype=torch.int32)
        m[:2] = torch.tensor([0, (1 << 23) - 1], device=DEV, dtype=torch.int32)
        Ns.append(((e + 127) << 23 | m).view(torch.float32))
    assert _sweep(q8, signed, torch.cat(Ns), Q=Q) == 0
