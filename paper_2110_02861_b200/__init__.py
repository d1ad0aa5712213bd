"""B200-native (sm_100a) block-wise dynamic 8-bit optimizer step (Dettmers et al. 2021,
arXiv 2110.02861).

The hot path lives in ``csrc/`` (CUDA kernels behind the C ABI ``include/q8.h``, built
into ``libq8.so``); this package is the thin Python binding plus the torch-facing
optimizer classes and the ZeRO-1 sharding wrapper.  There is no CPU fallback.
"""
from ._binding import (BLOCKSIZE, MAX_TENSORS_PER_LAUNCH, Q8Error, TensorList, create_dynamic_codebook,
                       create_linear_codebook, dequantize_blockwise, dequantize_tensorwise, hparams, nblocks,
                       optim8bit_step, optim8bit_step_multi, quantize_blockwise, quantize_blockwise_dynamic,
                       quantize_tensorwise, version)

__all__ = [
    "BLOCKSIZE", "MAX_TENSORS_PER_LAUNCH", "Q8Error", "TensorList", "create_dynamic_codebook",
    "create_linear_codebook", "dequantize_tensorwise", "quantize_tensorwise",
    "dequantize_blockwise", "hparams", "nblocks", "optim8bit_step", "optim8bit_step_multi", "quantize_blockwise",
    "quantize_blockwise_dynamic", "version",
]
from ._binding import layerwise_workspace_bytes, optim8bit_step_layerwise, optim32bit_step_multi  # noqa: E402
from ._binding import count_nonfinite, create_quantile_codebook, estimate_quantiles, quantiles_workspace_bytes  # noqa: E402
from ._binding import Plan, step_scalars, step_scalars_device  # noqa: E402
from .modules import StableEmbedding  # noqa: E402
from .optim import LAMB8bit, LARS8bit, Adam8bit, AdamW8bit, Momentum8bit, state_bytes  # noqa: E402
from .zero import Zero1Optimizer8bit, ZeroFusedOptimizer8bit, padded_numel, shard_range  # noqa: E402

__all__ += ["Plan", "step_scalars", "step_scalars_device", "count_nonfinite", "create_quantile_codebook", "estimate_quantiles", "quantiles_workspace_bytes",
            "layerwise_workspace_bytes", "optim8bit_step_layerwise", "LAMB8bit", "LARS8bit",
            "optim32bit_step_multi", "StableEmbedding", "Adam8bit", "AdamW8bit", "Momentum8bit", "state_bytes", "Zero1Optimizer8bit", "ZeroFusedOptimizer8bit", "padded_numel",
            "shard_range"]
