"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds NO arithmetic of the method (no codebook, no quantization, no
optimizer update).  It only draws seeded random numbers and describes workload
shapes, so both sides of every parity test start from identical bytes.

Input recipe, after SURVEY.md 8(d-2) and the paper's
runtime benchmark "a large sample of a normal distribution" (App. E):
  * params      p ~ N(0, 0.02^2)            (seed = base seed)
  * gradients   g ~ N(0, 1e-3^2), fresh per step (seed = 1000 + step), optional
                outliers: a fraction of elements multiplied by 100 ("outlier")
  * 8-bit state either zero (the valid initial state, Eq.2 "r_0 = m_0 = 0") or
                random codes with per-block absmax drawn from |N(0, scale^2)|
Shapes: GPT-2 medium / XL flat buffers, ResNet-50 tensor
list (161 tensors), T5-11B flat buffer.
"""
from __future__ import annotations

import math

import numpy as np
import torch

BLOCK = 2048

# ----------------------------------------------------------------------------- shapes


def gpt2_shapes(d: int, n_layer: int, vocab: int = 50257, ctx: int = 1024):
    shapes = [(vocab, d), (ctx, d)]
    for _ in range(n_layer):
        shapes += [(d,), (d,), (d, 3 * d), (3 * d,), (d, d), (d,), (d,), (d,), (d, 4 * d), (4 * d,),
                   (4 * d, d), (d,)]
    shapes += [(d,), (d,)]
    return shapes


def resnet50_shapes():
    shapes = [(64, 3, 7, 7), (64,), (64,)]
    inplanes = 64
    for width, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for bi in range(blocks):
            shapes += [(width, inplanes if bi == 0 else width * 4, 1, 1), (width,), (width,)]
            shapes += [(width, width, 3, 3), (width,), (width,)]
            shapes += [(width * 4, width, 1, 1), (width * 4,), (width * 4,)]
            if bi == 0:
                shapes += [(width * 4, inplanes, 1, 1), (width * 4,), (width * 4,)]
            inplanes = width * 4
        # (first block of each stage owns the downsample branch)
    shapes += [(1000, 2048), (1000,)]
    return shapes


def t5_11b_shapes(d=1024, d_ff=65536, inner=16384, n_layer=24, vocab=32128):
    shapes = [(vocab, d)]
    for _ in range(n_layer):  # encoder
        shapes += [(d, inner), (d, inner), (d, inner), (inner, d), (d,), (d, d_ff), (d_ff, d), (d,)]
    for _ in range(n_layer):  # decoder: self-attn, cross-attn, ffn
        shapes += [(d, inner), (d, inner), (d, inner), (inner, d), (d,)]
        shapes += [(d, inner), (d, inner), (d, inner), (inner, d), (d,)]
        shapes += [(d, d_ff), (d_ff, d), (d,)]
    shapes += [(d,), (d,), (32, 128), (32, 128)]
    return shapes


def numel(shape) -> int:
    return int(math.prod(shape))


WORKLOADS = {
    # name: (kind, grad dtype, shapes-or-n, description)  -- BASELINE.json configs
    "cfg1_1m": dict(kind="adam", grad_dtype="float32", n=1 << 20,
                    desc="codec round-trip + 10 steps 8-bit Adam, one flat 1M fp32 tensor"),
    "cfg2_gpt2_medium": dict(kind="adam", grad_dtype="float16", shapes=gpt2_shapes(1024, 24),
                             desc="8-bit Adam, 355M GPT-2-medium flat buffer, fp16 grads"),
    "cfg3_resnet50": dict(kind="momentum", grad_dtype="float16", shapes=resnet50_shapes(), multi=True,
                          desc="8-bit Momentum, ResNet-50 tensor list, multi-tensor launch"),
    "cfg4_gpt2_xl": dict(kind="adamw", grad_dtype="bfloat16", shapes=gpt2_shapes(1600, 48),
                         desc="8-bit AdamW, 1.5B GPT-2-XL flat buffer, bf16 grads"),
    "cfg5_t5_11b": dict(kind="adam", grad_dtype="bfloat16", shapes=t5_11b_shapes(),
                        desc="8-bit Adam, 11B T5-shaped flat buffer, ZeRO-1 over 8 GPUs"),
    # SURVEY 8(f) row 3 (T5 P:366-367): layer-wise optimizers over real layer lists (one trust
    # ratio per tensor), measured with the same bench contract
    "lamb_gpt2_xl": dict(kind="lamb", grad_dtype="bfloat16", shapes=gpt2_shapes(1600, 48), layerwise=True,
                         desc="8-bit LAMB, GPT-2-XL 580-tensor layer list, bf16 grads"),
    # the user-facing torch.optim API ("two-line change", P:7) over a real parameter list
    "optim_api_gpt2_xl": dict(kind="adamw", grad_dtype="bfloat16", shapes=gpt2_shapes(1600, 48), optim_api=True,
                              desc="AdamW8bit.step() over GPT-2-XL's 580 parameter tensors, bf16 grads"),
    # SURVEY 8(f) row 4 (App G): SRAM-Quantiles over a GPT-2-XL-sized fp32 buffer
    "quantiles_gpt2_xl": dict(kind="adamw", grad_dtype="float32", shapes=gpt2_shapes(1600, 48), quantiles=True,
                              desc="SRAM-Quantiles + Eq.5 codebook over a 1.5B fp32 GPT-2-XL-sized buffer"),
    # the stand-alone block-wise codec over a GPT-2-XL-sized fp32 buffer
    "codec_gpt2_xl": dict(kind="adam", grad_dtype="float32", shapes=gpt2_shapes(1600, 48), codec=True,
                          desc="block-wise quantize (dynamic and generic table) + dequantize, 1.5B fp32 buffer"),
    "lars_resnet50": dict(kind="lars", grad_dtype="float16", shapes=resnet50_shapes(), layerwise=True,
                          desc="8-bit LARS, ResNet-50 161-tensor layer list, fp16 grads"),
}

HPARAMS = {
    # SURVEY 8(d-2); second Adam set = the paper's sensitivity baseline
    "adam": dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, bias_correction=True),
    "adam_paper": dict(lr=0.0163, beta1=0.9, beta2=0.995, eps=1e-7, weight_decay=0.0, bias_correction=True),
    "adamw": dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, bias_correction=True),
    "momentum": dict(lr=0.1, beta1=0.9, beta2=0.0, eps=1e-8, weight_decay=1e-4, bias_correction=False),
    # layer-wise optimizers of T5: LAMB (You et al. 2020 defaults), LARS (You et al.
    # 2017: trust coefficient eta = 0.001, wd 5e-4, momentum 0.9)
    "lamb": dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01, bias_correction=True),
    "lars": dict(lr=0.1, beta1=0.9, beta2=0.0, eps=1e-8, weight_decay=5e-4, bias_correction=False,
                 trust_coefficient=0.001),
}


def workload_numel(name: str) -> int:
    w = WORKLOADS[name]
    return w["n"] if "n" in w else sum(numel(s) for s in w["shapes"])


# ----------------------------------------------------------------------------- draws

_TORCH_DT = {"float32": torch.float32, "float16": torch.float16, "bfloat16": torch.bfloat16}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def params(n: int, seed: int = 0, device="cpu", std: float = 0.02) -> torch.Tensor:
    """p ~ N(0, std^2), float32."""
    return torch.randn(n, generator=_gen(seed, device), device=device, dtype=torch.float32).mul_(std)


def grads(n: int, step: int, seed: int = 0, dtype: str = "float32", device="cpu", std: float = 1e-3,
          outlier_frac: float = 0.0, outlier_scale: float = 100.0) -> torch.Tensor:
    """g ~ N(0, std^2) drawn in float32 then cast to dtype; a seeded `outlier_frac` of the
    elements is multiplied by `outlier_scale` before the cast."""
    gen = _gen(1000 + 7919 * seed + step, device)
    g = torch.randn(n, generator=gen, device=device, dtype=torch.float32).mul_(std)
    if outlier_frac > 0:
        k = max(1, int(n * outlier_frac))
        idx = torch.randint(0, n, (k,), generator=gen, device=device)
        g[idx] *= outlier_scale
    return g.to(_TORCH_DT[dtype])


def zero_state(n: int, blocksize: int = BLOCK, device="cpu"):
    nb = (n + blocksize - 1) // blocksize
    return (torch.zeros(n, dtype=torch.uint8, device=device), torch.zeros(nb, dtype=torch.float32, device=device))


def random_state(n: int, seed: int, blocksize: int = BLOCK, device="cpu", scale: float = 1e-3,
                 low: int = 0, high: int = 256):
    """Random 8-bit state: codes uniform in [low, high), absmax ~ |N(0, scale^2)| per block."""
    nb = (n + blocksize - 1) // blocksize
    gen = _gen(5000 + seed, device)
    codes = torch.randint(low, high, (n,), generator=gen, device=device, dtype=torch.int32).to(torch.uint8)
    absmax = torch.randn(nb, generator=gen, device=device, dtype=torch.float32).abs_().mul_(scale)
    return codes, absmax


def uniform(n: int, seed: int, lo: float = -1.0, hi: float = 1.0, device="cpu") -> torch.Tensor:
    return torch.rand(n, generator=_gen(seed, device), device=device, dtype=torch.float32) * (hi - lo) + lo


def to_f32_numpy(t: torch.Tensor) -> np.ndarray:
    """Exact widening of a float16/bfloat16/float32 tensor to a float32 numpy array."""
    return t.detach().to("cpu").to(torch.float32).numpy()
