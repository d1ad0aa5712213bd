"""GPU tests of the fused ZeRO-1 step over peer memory (reading Z1).

* one rank: the fused kernel equals the plain fused step bit for bit (g / 1 = g);
* two ranks as two processes sharing cuda:0 (CUDA IPC mappings, flag barriers in each rank's
  signal pad, 74 CTAs per rank so both grids are resident): after every step both ranks' full
  parameter buffers and each rank's shard states equal the oracle: g = (g_0 + g_1) / 2 in
  binary32, then the 8-bit step of each shard (oracle.optim8bit_step)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kind,gdt", [("adamw", "bfloat16"), ("momentum", "float16"), ("adam", "float32")])
def test_single_rank_equals_plain_step(kind, gdt):
    import paper_2110_02861_b200 as q8
    n = 9 * 2048 + 300
    hp = dict(synth.HPARAMS[kind])
    zo = q8.ZeroFusedOptimizer8bit(n, kind=kind, grad_dtype=getattr(torch, gdt), device="cuda", **hp)
    p = synth.params(n).cuda()
    zo.params[:n] = p
    s1, a1 = synth.zero_state(n, device="cuda")
    s2, a2 = synth.zero_state(n, device="cuda")
    for t in range(1, 4):
        g = synth.grads(n, step=t, dtype=gdt).cuda()
        zo.grads[:n] = g
        zo.step()
        q8.optim8bit_step(kind, p, g, s1, s2, a1, a2, step=t, **hp)
    torch.cuda.synchronize()
    assert torch.equal(zo.params[:n].view(torch.int32), p.view(torch.int32))
    assert torch.equal(zo.s1[:n], s1) and torch.equal(zo.absmax1[:a1.numel()], a1)
    if kind != "momentum":
        assert torch.equal(zo.s2[:n], s2) and torch.equal(zo.absmax2[:a2.numel()], a2)
    assert torch.count_nonzero(zo.params[n:]) == 0


def _run_ranks(tmp_path, kind, gdt, world, mode, ctas):
    n, steps = 13 * 2048 + 777, 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + (os.getpid() % 300)),
           os.path.join(ROOT, "tests", "_zero_fused_worker.py"), str(tmp_path), str(n), kind, gdt, str(steps),
           str(ctas), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    _check_against_oracle(tmp_path, kind, gdt, world, n, steps)


@pytest.mark.parametrize("kind,gdt", [("adamw", "bfloat16"), ("momentum", "float32")])
def test_two_ranks_sharing_one_gpu(tmp_path, kind, gdt):
    _run_ranks(tmp_path, kind, gdt, 2, "shared", 74)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NVLS multicast needs one GPU per rank (>= 2 GPUs)")
@pytest.mark.parametrize("kind,gdt", [("adamw", "bfloat16"), ("adam", "float16")])
def test_nvls_multicast_all_gather(tmp_path, kind, gdt):
    """One rank per GPU (NCCL), buffers in torch symmetric memory, the all-gather as multimem.st
    through NVSwitch: bit-exact against the oracle like the peer-store path (reading Z1)."""
    _run_ranks(tmp_path, kind, gdt, min(4, torch.cuda.device_count()), "nvls", 0)


def _check_against_oracle(tmp_path, kind, gdt, world, n, steps):
    hp = dict(synth.HPARAMS[kind])
    B = 2048
    unit = world * B
    n_pad = (n + unit - 1) // unit * unit
    shard = n_pad // world
    p = np.zeros(n_pad, np.float32)
    p[:n] = synth.params(n, seed=3).numpy()
    st = [dict(s1=np.zeros(shard, np.uint8), s2=np.zeros(shard, np.uint8), a1=np.zeros(shard // B, np.float32),
               a2=np.zeros(shard // B, np.float32)) for _ in range(world)]
    for t in range(1, steps + 1):
        gs = []
        for rk in range(world):
            g = np.zeros(n_pad, np.float32)
            g[:n] = synth.to_f32_numpy(synth.grads(n, step=t, seed=50 + rk, dtype=gdt))
            gs.append(g)
        acc = gs[0].copy()
        for g in gs[1:]:
            acc = (acc + g).astype(np.float32)       # binary32 adds in rank order (Z1)
        acc = (acc / np.float32(world)).astype(np.float32)
        for rk in range(world):
            lo = rk * shard
            ps = p[lo:lo + shard].copy()
            s = st[rk]
            oracle.optim8bit_step(kind, ps, acc[lo:lo + shard], s["s1"], s["s2"], s["a1"], s["a2"], step=t, **hp)
            p[lo:lo + shard] = ps
        for rk in range(world):
            got = np.load(tmp_path / f"r{rk}_t{t}.npz")
            assert np.array_equal(got["p"].view(np.uint32), p.view(np.uint32)), (t, rk)
            assert np.array_equal(got["s1"], st[rk]["s1"]) and np.array_equal(got["a1"], st[rk]["a1"])
            if kind != "momentum":
                assert np.array_equal(got["s2"], st[rk]["s2"]) and np.array_equal(got["a2"], st[rk]["a2"])
