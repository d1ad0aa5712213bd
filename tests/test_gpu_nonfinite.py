"""GPU check of q8_count_nonfinite (SURVEY 5 failure detection: non-finite gradients are out of the
step's contract, G13): the count equals numpy's count of non-finite values, for every gradient dtype,
at sizes with vector tails, with NaN, +inf, -inf and the largest finite values mixed in."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

DT = {"float32": torch.float32, "float16": torch.float16, "bfloat16": torch.bfloat16}


@pytest.fixture(scope="module")
def q8():
    import paper_2110_02861_b200 as m
    return m


@pytest.mark.parametrize("dtype", list(DT))
@pytest.mark.parametrize("n", [1, 7, 9, 4099, 1_000_003])
def test_count_matches_numpy(q8, dtype, n):
    g = synth.grads(n, step=1, dtype=dtype, std=1.0)
    gen = torch.Generator().manual_seed(n)
    k = max(1, n // 1000)
    idx = torch.randint(0, n, (k,), generator=gen)
    vals = torch.tensor([float("nan"), float("inf"), -float("inf")])[torch.randint(0, 3, (k,), generator=gen)]
    g[idx] = vals.to(g.dtype)
    g[torch.randint(0, n, (k,), generator=gen)] = torch.finfo(g.dtype).max  # finite extremes stay finite
    want = int((~np.isfinite(g.to(torch.float32).numpy())).sum())
    got = int(q8.count_nonfinite(g.cuda()).item())
    assert got == want


@pytest.mark.parametrize("dtype", list(DT))
def test_clean_and_empty(q8, dtype):
    g = synth.grads(123_457, step=2, dtype=dtype).cuda()
    assert int(q8.count_nonfinite(g).item()) == 0
    assert int(q8.count_nonfinite(g[:0]).item()) == 0
