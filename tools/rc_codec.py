"""Sanitizer helper: one caller-table block-wise quantize long enough for the per-CTA bucket table (>= 16 blocks
per CTA), checked against the oracle (usage: rc_codec.py [blocks])."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2110_02861_b200 as q8  # noqa: E402
import synth  # noqa: E402
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 16 * torch.cuda.get_device_properties(0).multi_processor_count
rng = np.random.default_rng(3)
Q = oracle.quantile_codebook(oracle.exact_quantiles(rng.standard_normal(1 << 16).astype(np.float32)))
x = synth.params(nb * 2048, seed=9)
a, c = q8.quantize_blockwise(torch.from_numpy(Q).cuda(), x.cuda())
a_r, c_r = oracle.quantize_blockwise(Q, x.numpy())
assert np.array_equal(c.cpu().numpy(), c_r) and np.array_equal(a.cpu().numpy().view(np.uint32), a_r.view(np.uint32))
print("ok", nb, "blocks")
