"""The Stable Embedding layer (S3.3; App. C).

"We initialize the Stable Embedding Layer with Xavier uniform initialization and apply layer
normalization before adding position embeddings ... we find that the stability of training
improves significantly if we use 32-bit optimizer states for the embedding layers."  The
module marks its weight so that the 8-bit optimizers of this package keep that tensor's states
in 32 bits (``q8_optim32bit_step_multi``)."""
from __future__ import annotations

import torch
import torch.nn.functional as F


class StableEmbedding(torch.nn.Embedding):
    def __init__(self, num_embeddings: int, embedding_dim: int, padding_idx=None, max_norm=None, norm_type=2.0,
                 scale_grad_by_freq=False, sparse=False, device=None, dtype=None):
        super().__init__(num_embeddings, embedding_dim, padding_idx, max_norm, norm_type, scale_grad_by_freq, sparse,
                         device=device, dtype=dtype)
        self.norm = torch.nn.LayerNorm(embedding_dim, device=device)
        self.weight._q8_optim_bits = 32   # 32-bit optimizer states for this layer

    def reset_parameters(self) -> None:
        # Xavier uniform (Glorot): U(-b, b), b = sqrt(6 / (fan_in + fan_out)) = sqrt(6 / (V + D))
        torch.nn.init.xavier_uniform_(self.weight)
        self._fill_padding_idx_with_zero()

    def forward(self, input: torch.Tensor) -> torch.Tensor:
        emb = F.embedding(input, self.weight, self.padding_idx, self.max_norm, self.norm_type,
                          self.scale_grad_by_freq, self.sparse)
        return self.norm(emb.to(self.norm.weight.dtype))
