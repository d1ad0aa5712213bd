"""ZeRO-1 plumbing on CPU ranks (gloo, world size 2): block-aligned padding and shard ranges,
reduce-scatter -> shard step -> all-gather, and equivalence of the sharded result with one
unsharded step on the same reduced gradient (blocks are independent).

The per-shard step is injected (the CUDA kernel needs a GPU); here it is the oracle, which is
allowed in tests only.  The collective sequence and shard bookkeeping are the product code."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2110_02861_b200 import zero

HP = synth.HPARAMS["adamw"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def oracle_step(kind):
    def fn(p, g, s1, s2, a1, a2, step):
        oracle.optim8bit_step(kind, p.numpy(), synth.to_f32_numpy(g), s1.numpy(), None if s2 is None else s2.numpy(),
                              a1.numpy(), None if a2 is None else a2.numpy(), step=step, **HP)
    return fn


def _worker(rank, world, port, n, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        zo = zero.Zero1Optimizer8bit(n, kind="adamw", grad_dtype=torch.bfloat16, device="cpu",
                                     step_fn=oracle_step("adamw"), **HP)
        assert zo.n_pad % (world * 2048) == 0 and zo.n_pad >= n
        assert (zo.hi - zo.lo) == zo.n_pad // world and zo.lo % 2048 == 0
        zo.params[:n] = synth.params(n, seed=3)
        full_ref = zo.params.clone()
        s1r = torch.zeros(zo.n_pad, dtype=torch.uint8)
        s2r = torch.zeros(zo.n_pad, dtype=torch.uint8)
        a1r = torch.zeros(zo.n_pad // 2048)
        a2r = torch.zeros(zo.n_pad // 2048)
        ok = True
        for t in range(1, steps + 1):
            zo.grads.zero_()
            zo.grads[:n] = synth.grads(n, step=t, seed=rank, dtype="bfloat16")   # rank-local grads
            zo.reduce_scatter()
            # the reduced gradient, gathered, drives the unsharded reference step
            g_full = torch.empty(zo.n_pad, dtype=torch.bfloat16)
            dist.all_gather_into_tensor(g_full, zo.g_shard)
            zo.shard_step()
            zo.all_gather()
            oracle.optim8bit_step("adamw", full_ref.numpy(), synth.to_f32_numpy(g_full), s1r.numpy(), s2r.numpy(),
                                  a1r.numpy(), a2r.numpy(), step=t, **HP)
            ok &= bool(torch.equal(zo.params.view(torch.int32), full_ref.view(torch.int32)))
            ok &= bool(torch.equal(zo.s1, s1r[zo.lo:zo.hi])) and bool(torch.equal(zo.s2, s2r[zo.lo:zo.hi]))
            ok &= bool(torch.equal(zo.absmax1, a1r[zo.lo // 2048:zo.hi // 2048]))
            # padding stays neutral
            ok &= bool(torch.all(zo.params[n:] == 0))
        out[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [5 * 2048 + 333, 4 * 2048])
def test_zero1_two_ranks_equals_unsharded(n):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, 3, out), nprocs=world, join=True)
    assert out[0] and out[1]


def test_padding_and_shards():
    for n, w in [(1, 1), (2048, 2), (2049, 2), (1_557_611_200, 8), (11_307_321_344, 8)]:
        npad = zero.padded_numel(n, w)
        assert npad >= n and npad % (w * 2048) == 0 and npad - n < w * 2048
        ranges = [zero.shard_range(npad, w, r) for r in range(w)]
        assert ranges[0][0] == 0 and ranges[-1][1] == npad
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert all((hi - lo) % 2048 == 0 for lo, hi in ranges)
