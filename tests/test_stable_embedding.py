"""StableEmbedding (S3.3) on CPU: Xavier-uniform support and variance, layer-normalized
output, and the 32-bit optimizer-state marker on its weight."""
import math

import torch

from paper_2110_02861_b200 import StableEmbedding


def test_init_and_forward():
    torch.manual_seed(0)
    V, D = 1000, 64
    emb = StableEmbedding(V, D)
    b = math.sqrt(6.0 / (V + D))                     # Xavier uniform bound
    w = emb.weight.detach()
    assert float(w.abs().max()) <= b
    assert abs(float(w.var()) - b * b / 3) < 0.05 * b * b / 3   # U(-b, b) variance b^2/3
    y = emb(torch.randint(0, V, (8, 32)))
    assert y.shape == (8, 32, D)
    assert float(y.mean(-1).abs().max()) < 1e-3       # LayerNorm: per position mean 0
    assert abs(float(y.var(-1, unbiased=False).mean()) - 1.0) < 1e-2   # and variance ~1
    assert getattr(emb.weight, "_q8_optim_bits") == 32
