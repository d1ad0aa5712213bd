"""GPU parity for SRAM-Quantiles (App G) and the quantile data type (Eq.5, App F.2),
through the C ABI, against the CPU oracle.

Bar (reading Q4): the chunk quantiles are order statistics (exact); the mean over
chunks is accumulated in binary64 in a different order than the oracle's, so the fp32 results may
differ by the reordering bound 2*C*2^-53*max|x| plus one fp32 ulp of the final rounding.  Where the
binary64 sums are exact (one chunk; small-integer data) the results must be bit-identical, and so
must the Eq.5 codebooks built from them.  Inputs from synth (seeded) or closed forms; expected
values from oracle/ only."""
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


def ulp32(v):
    v = np.abs(np.asarray(v, np.float32))
    return np.spacing(np.maximum(v, np.float32(np.finfo(np.float32).tiny))).astype(np.float64)


def assert_close_q4(gpu, ref, n, xmax, what=""):
    chunks = (n + 4095) // 4096
    tol = ulp32(ref) + 2.0 * chunks * 2.0 ** -53 * float(xmax)
    diff = np.abs(gpu.astype(np.float64) - ref.astype(np.float64))
    bad = np.nonzero(diff > tol)[0]
    assert bad.size == 0, f"{what}: {bad.size} quantiles outside the Q4 bound, e.g. j={bad[:4]} gpu={gpu[bad[:4]]} ref={ref[bad[:4]]}"
    return int((gpu.view(np.uint32) != ref.view(np.uint32)).sum())


SIZES = [1, 2, 17, 255, 4095, 4096, 4097, 3 * 4096 + 5, 100_003, 1_000_000, 1 << 20]


@pytest.mark.parametrize("n", SIZES)
def test_sram_quantiles_gaussian(q8, n):
    x = synth.params(n, seed=n, std=1.0)
    q_g = q8.estimate_quantiles(x.to(DEV)).cpu().numpy()
    q_r = oracle.sram_quantiles(x.numpy())
    if n <= 4096:  # one chunk: the estimate is an order statistic, bit for bit
        np.testing.assert_array_equal(q_g.view(np.uint32), q_r.view(np.uint32))
    else:
        assert_close_q4(q_g, q_r, n, x.abs().max().item(), f"n={n}")


@pytest.mark.parametrize("n", [4096 * 7 + 1000, 1 << 20])
def test_sram_quantiles_integer_data_bit_exact(q8, n):
    # small integers with many ties: every binary64 sum is exact, so results are bit-identical
    g = torch.Generator().manual_seed(n)
    x = torch.randint(-50, 50, (n,), generator=g).to(torch.float32)
    q_g = q8.estimate_quantiles(x.to(DEV)).cpu().numpy()
    q_r = oracle.sram_quantiles(x.numpy())
    np.testing.assert_array_equal(q_g.view(np.uint32), q_r.view(np.uint32))


@pytest.mark.parametrize("case", ["sorted", "reversed", "constant", "zeros_signed", "wide_exponents", "tiny_tail"])
def test_sram_quantiles_edge_inputs(q8, case):
    n = 4096 * 5 + 3
    x = synth.params(n, seed=3, std=1.0)
    if case == "sorted":
        x = torch.sort(x).values
    elif case == "reversed":
        x = torch.sort(x, descending=True).values
    elif case == "constant":
        x = torch.full((n,), -2.5)
    elif case == "zeros_signed":  # -0 and +0 mixed with a few values
        x = torch.zeros(n)
        x[::3] = -0.0
        x[::101] = 1.0
    elif case == "wide_exponents":  # magnitudes over ~70 binades
        x = x.sign() * torch.exp2(synth.uniform(n, seed=4, lo=-60, hi=10))
    elif case == "tiny_tail":  # the last chunk holds 3 elements
        x[-3:] = torch.tensor([1e6, -1e6, 0.5])
    q_g = q8.estimate_quantiles(x.contiguous().to(DEV)).cpu().numpy()
    q_r = oracle.sram_quantiles(x.numpy())
    assert_close_q4(q_g, q_r, n, x.abs().max().item(), case)
    assert np.all(np.diff(q_g) >= 0)


@pytest.mark.parametrize("n", [300, 4096, 4096 * 3])
def test_device_codebook_matches_oracle(q8, n):
    # one chunk or integer data: the quantiles are bit-identical, so the Eq.5 codebooks must be too
    if n <= 4096:
        x = synth.params(n, seed=9, std=0.5)
    else:
        x = torch.randint(-1000, 1000, (n,), generator=torch.Generator().manual_seed(1)).to(torch.float32) / 64
    q_g, c_g = q8.estimate_quantiles(x.to(DEV), with_codebook=True)
    q_r = oracle.sram_quantiles(x.numpy())
    np.testing.assert_array_equal(q_g.cpu().numpy().view(np.uint32), q_r.view(np.uint32))
    c_r = oracle.quantile_codebook(q_r)
    np.testing.assert_array_equal(c_g.cpu().numpy().view(np.uint32), c_r.view(np.uint32))


def test_quantile_quantization_end_to_end(q8):
    # quantile quantization (App F.2): the oracle's quantile codebook drives the GPU block codec,
    # bit-exact against the oracle codec with the same table
    n = 200_003
    x = synth.params(n, seed=21, std=1.0)
    code = oracle.quantile_codebook(oracle.sram_quantiles(x.numpy()))
    a_g, c_g = q8.quantize_blockwise(torch.from_numpy(code).to(DEV), x.to(DEV))
    a_r, c_r = oracle.quantize_blockwise(code, x.numpy())
    np.testing.assert_array_equal(a_g.cpu().numpy().view(np.uint32), a_r.view(np.uint32))
    np.testing.assert_array_equal(c_g.cpu().numpy(), c_r)


def test_quantile_type_is_near_minimum_entropy(q8):
    # "the quantized outputs take the value of each of the 2^k different bit representations
    # equally often": tensor-wise quantization of N(0,1) data with its own SRAM-Quantiles
    # codebook uses every code about n/256 times
    n = 4096 * 256
    x = synth.params(n, seed=5, std=1.0).to(DEV)
    q, code = q8.estimate_quantiles(x, with_codebook=True)
    qd = q.double()
    M = ((qd[:-1] + qd[1:]) * 0.5).abs().max().float()   # the scale the codebook was normalized by
    _, codes = q8.quantize_tensorwise(code, x.clamp(-M, M).contiguous())  # so that N = M
    hist = torch.bincount(codes.long(), minlength=256).cpu().numpy()
    interior = hist[2:254]
    assert interior.min() > 0.8 * n / 256 and interior.max() < 1.2 * n / 256, (interior.min(), interior.max())


@pytest.mark.slow
def test_sram_quantiles_full_size_closed_form(q8):
    # GPT-2-XL-sized buffer (1,557,611,200 elements, 380,276 chunks, the bench workload): chunk c is
    # a permutation of 0..4095 plus (c mod 7); the chunk quantiles are floor(j*4096/257) + (c mod 7)
    # exactly, so the estimate is floor(j*4096/257) + mean(c mod 7) (the last chunk is short: m = 1600)
    n = synth.workload_numel("cfg4_gpt2_xl")
    C = (n + 4095) // 4096
    last = n - (C - 1) * 4096
    g = torch.Generator(device=DEV).manual_seed(0)
    perm = torch.randperm(4096, generator=g, device=DEV).to(torch.float32)
    x = torch.empty(C * 4096, device=DEV)
    xv = x.view(C, 4096)
    xv.copy_(perm.expand(C, 4096))
    xv.add_((torch.arange(C, device=DEV) % 7).to(torch.float32)[:, None])
    x = x[:n]
    q_g = q8.estimate_quantiles(x).cpu().numpy().astype(np.float64)
    off = np.arange(C) % 7
    base_last = np.sort(perm.cpu().numpy()[:last])  # the short chunk: its own order statistics
    want = np.empty(257)
    for j in range(257):
        full = (C - 1) * ((j * 4096) // 257) + off[:-1].sum()
        want[j] = (full + base_last[(j * last) // 257] + off[-1]) / C
    np.testing.assert_array_equal(q_g.astype(np.float32), want.astype(np.float32))
    del x, xv
