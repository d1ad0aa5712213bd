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
    bits = base.view(torch.int32)
    # step |x| by d ulps in the direction of increasing value (negative values: bits move the other way)
    step = torch.where(base < 0, -d[None, :], d[None, :])
    stepped = (bits + step).view(torch.float32)
    x[:, 1:2041] = torch.where(base == 0, base, stepped)
    x[:, 2041] = -N
    x[:, 2042] = N
    return x


def _expected(x, N, bnd64):
    y = (x.to(torch.float64) / N.to(torch.float64)[:, None]).to(torch.float32).to(torch.float64)
    return torch.searchsorted(bnd64, y.reshape(-1), right=True).reshape(x.shape)


def _sweep(q8, signed, N, chunk=1 << 17):
    Q = oracle.dynamic_codebook(signed)
    bnd = _boundaries(Q)
    bnd64 = torch.from_numpy(bnd).to(DEV)
    bnd32 = torch.from_numpy(bnd.astype(np.float32)).to(DEV)
    bad = 0
    for s in range(0, N.numel(), chunk):
        Nc = N[s:s + chunk]
        x = _blocks(Nc, bnd32)
        if not signed:
            x = x.abs()    # unsigned table: non-negative states; boundaries are all >= 0
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
