"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times: one fused
step over the whole flat buffer on the GPU, then the oracle recomputes sampled blocks one by one
(blocks are independent) and every sampled output must match bit for bit.  Sampled: 48
random blocks, the first, and the last (ragged) block."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda"
B = 2048


@pytest.mark.parametrize("workload,steps", [("cfg4_gpt2_xl", 2), ("cfg2_gpt2_medium", 2)])
def test_full_size_sampled_blocks(workload, steps):
    import paper_2110_02861_b200 as q8
    w = synth.WORKLOADS[workload]
    kind, gdt = w["kind"], w["grad_dtype"]
    hp = dict(synth.HPARAMS[kind])
    n = synth.workload_numel(workload)
    nb = (n + B - 1) // B
    p = synth.params(n, seed=21, device=DEV)
    s1, a1 = synth.random_state(n, seed=22, device=DEV, scale=1e-3)
    s2, a2 = synth.random_state(n, seed=23, device=DEV, scale=1e-6)
    rng = np.random.default_rng(7)
    blocks = sorted(set([0, nb - 1] + rng.integers(0, nb, 48).tolist()))

    def take(t, b):
        return t[b * B:min((b + 1) * B, n)].cpu().numpy().copy()

    ref = {b: dict(p=take(p, b), s1=take(s1, b), s2=take(s2, b), a1=a1[b:b + 1].cpu().numpy().copy(),
                   a2=a2[b:b + 1].cpu().numpy().copy()) for b in blocks}
    for t in range(1, steps + 1):
        g = synth.grads(n, step=t, seed=5, dtype=gdt, device=DEV)
        q8.optim8bit_step(kind, p, g, s1, s2, a1, a2, step=t, **hp)
        for b, r in ref.items():
            gb = synth.to_f32_numpy(g[b * B:min((b + 1) * B, n)])
            oracle.optim8bit_step(kind, r["p"], gb, r["s1"], r["s2"], r["a1"], r["a2"], step=t, **hp)
        del g
    torch.cuda.synchronize()
    for b, r in ref.items():
        assert np.array_equal(take(p, b).view(np.uint32), r["p"].view(np.uint32)), f"p block {b}"
        assert np.array_equal(take(s1, b), r["s1"]), f"s1 block {b}"
        assert np.array_equal(take(s2, b), r["s2"]), f"s2 block {b}"
        assert a1[b].item() == r["a1"][0] and a2[b].item() == r["a2"][0], f"absmax block {b}"


def test_full_size_momentum_multi_tensor_gpt2_medium_list():
    """BASELINE config 3's multi-tensor path at a larger tensor list (GPT-2-medium, 292 tensors,
    fp16 grads, Momentum): one launch per <= 384 tensors; every tensor's first and last block."""
    import paper_2110_02861_b200 as q8
    hp = dict(synth.HPARAMS["momentum"])
    shapes = synth.gpt2_shapes(1024, 24)
    ents, refs = [], []
    for i, sh in enumerate(shapes):
        n = synth.numel(sh)
        p = synth.params(n, seed=300 + i, device=DEV)
        g = synth.grads(n, step=1, seed=300 + i, dtype="float16", device=DEV)
        s1, a1 = synth.random_state(n, seed=400 + i, device=DEV)
        ents.append((p, g, s1, None, a1, None))
        nb = (n + B - 1) // B
        sel = sorted({0, nb - 1})
        refs.append({b: (p[b * B:min((b + 1) * B, n)].cpu().numpy().copy(),
                         synth.to_f32_numpy(g[b * B:min((b + 1) * B, n)]),
                         s1[b * B:min((b + 1) * B, n)].cpu().numpy().copy(), a1[b:b + 1].cpu().numpy().copy())
                     for b in sel})
    q8.optim8bit_step_multi("momentum", ents, step=3, **hp)
    torch.cuda.synchronize()
    for (p, g, s1, _, a1, _), rb in zip(ents, refs):
        n = p.numel()
        for b, (rp, rg, rs, ra) in rb.items():
            oracle.optim8bit_step("momentum", rp, rg, rs, None, ra, None, step=3, **hp)
            assert np.array_equal(p[b * B:min((b + 1) * B, n)].cpu().numpy().view(np.uint32), rp.view(np.uint32))
            assert np.array_equal(s1[b * B:min((b + 1) * B, n)].cpu().numpy(), rs)
            assert a1[b].item() == ra[0]


def test_full_size_t5_11b_beyond_2_32_elements():
    """BASELINE config 5 unsharded on one GPU: 11,307,321,344 parameters (> 2^32 elements: the 64-bit
    element offsets of the kernel), 8-bit Adam, bf16 gradients, two steps from the zero state; sampled
    blocks on both sides of 2^31 and 2^32 elements, random blocks, and the ragged last block."""
    import paper_2110_02861_b200 as q8
    workload = "cfg5_t5_11b"
    kind = "adam"
    hp = dict(synth.HPARAMS[kind])
    n = synth.workload_numel(workload)
    assert n > 2 ** 32
    nb = (n + B - 1) // B
    free, _ = torch.cuda.mem_get_info()
    if free < n * 9.5:
        pytest.skip(f"needs ~{n * 9.5 / 2**30:.0f} GiB of device memory")
    p = torch.empty(n, dtype=torch.float32, device=DEV)
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    chunk = 1 << 28
    for k, lo in enumerate(range(0, n, chunk)):  # seeded chunks (no full-size fp32 temporary)
        hi = min(lo + chunk, n)
        p[lo:hi] = synth.params(hi - lo, seed=500 + k, device=DEV)
    s1, a1 = synth.zero_state(n, device=DEV)
    s2, a2 = synth.zero_state(n, device=DEV)
    rng = np.random.default_rng(11)
    edges = [(2 ** 31) // B - 1, (2 ** 31) // B, (2 ** 32) // B - 1, (2 ** 32) // B]
    blocks = sorted(set([0, nb - 1] + edges + rng.integers(0, nb, 24).tolist()))

    def take(t, b):
        return t[b * B:min((b + 1) * B, n)].cpu().numpy().copy()

    ref = {b: dict(p=take(p, b), s1=take(s1, b), s2=take(s2, b), a1=a1[b:b + 1].cpu().numpy().copy(),
                   a2=a2[b:b + 1].cpu().numpy().copy()) for b in blocks}
    for t in (1, 2):
        for k, lo in enumerate(range(0, n, chunk)):
            hi = min(lo + chunk, n)
            g[lo:hi] = synth.grads(hi - lo, step=t, seed=k, dtype="bfloat16", device=DEV)
        q8.optim8bit_step(kind, p, g, s1, s2, a1, a2, step=t, **hp)
        for b, r in ref.items():
            oracle.optim8bit_step(kind, r["p"], synth.to_f32_numpy(g[b * B:min((b + 1) * B, n)]), r["s1"], r["s2"],
                                  r["a1"], r["a2"], step=t, **hp)
    torch.cuda.synchronize()
    for b, r in ref.items():
        assert np.array_equal(take(p, b).view(np.uint32), r["p"].view(np.uint32)), f"p block {b}"
        assert np.array_equal(take(s1, b), r["s1"]), f"s1 block {b}"
        assert np.array_equal(take(s2, b), r["s2"]), f"s2 block {b}"
        assert a1[b].item() == r["a1"][0] and a2[b].item() == r["a2"][0], f"absmax block {b}"
    del p, g, s1, s2, a1, a2
    torch.cuda.empty_cache()
