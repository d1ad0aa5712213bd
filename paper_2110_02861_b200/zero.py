"""ZeRO-1 data parallelism for the 8-bit step (optimizer sharding is cited as
complementary in the paper, P:259 S6).

One process per GPU.  The flat fp32 parameter buffer is padded to a multiple of
``world * 2048`` elements (zero padding is neutral: zeros never raise a block's absmax and
padded p, g stay 0) and split on block boundaries, so every rank's shard is a whole number of
2048-element blocks (blocks are independent, P:110 -- the sharded result equals the
unsharded one bit for bit).  Each step:

  1. ``reduce_scatter_tensor`` of the full gradient buffer (NCCL over NVLink; op AVG)
  2. the fused 8-bit step on this rank's shard (its own 8-bit states only)
  3. ``all_gather_into_tensor`` of the updated parameter shards back into the full buffer.

``step_fn`` is the per-shard step; it defaults to the CUDA kernel and is injectable only
so the collective plumbing can be tested on CPU ranks (gloo).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _binding as B


def padded_numel(n: int, world: int, blocksize: int = B.BLOCKSIZE) -> int:
    unit = world * blocksize
    return (n + unit - 1) // unit * unit


def shard_range(n_padded: int, world: int, rank: int):
    shard = n_padded // world
    return rank * shard, (rank + 1) * shard


class Zero1Optimizer8bit:
    def __init__(self, n_params: int, kind: str = "adamw", grad_dtype=torch.bfloat16, device=None, group=None,
                 step_fn=None, state_device=None, **hparams):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.kind = kind
        self.n = n_params
        self.n_pad = padded_numel(n_params, self.world)
        self.lo, self.hi = shard_range(self.n_pad, self.world, self.rank)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        sdev = torch.device(state_device) if state_device is not None else dev
        self.params = torch.zeros(self.n_pad, dtype=torch.float32, device=dev)   # full replica
        self.grads = torch.zeros(self.n_pad, dtype=grad_dtype, device=dev)       # full local grads
        shard = self.hi - self.lo
        self.g_shard = torch.zeros(shard, dtype=grad_dtype, device=sdev)
        self.s1 = torch.zeros(shard, dtype=torch.uint8, device=sdev)
        self.absmax1 = torch.zeros(shard // B.BLOCKSIZE, dtype=torch.float32, device=sdev)
        two = kind != "momentum"
        self.s2 = torch.zeros(shard, dtype=torch.uint8, device=sdev) if two else None
        self.absmax2 = torch.zeros(shard // B.BLOCKSIZE, dtype=torch.float32, device=sdev) if two else None
        self.hp = dict(hparams)
        self.t = 0
        self.step_fn = step_fn or self._cuda_step

    @property
    def p_shard(self) -> torch.Tensor:
        return self.params[self.lo:self.hi]

    def _cuda_step(self, p, g, s1, s2, a1, a2, step):
        B.optim8bit_step(self.kind, p, g, s1, s2, a1, a2, step=step, **self.hp)

    def reduce_scatter(self):
        if not dist.is_initialized():
            self.g_shard.copy_(self.grads[self.lo:self.hi])
            return
        try:
            dist.reduce_scatter_tensor(self.g_shard, self.grads, op=dist.ReduceOp.AVG, group=self.group)
        except (RuntimeError, ValueError):  # backends without AVG reduce-scatter (gloo)
            dist.reduce_scatter_tensor(self.g_shard, self.grads, op=dist.ReduceOp.SUM, group=self.group)
            self.g_shard.div_(self.world)

    def all_gather(self):
        if dist.is_initialized():
            dist.all_gather_into_tensor(self.params, self.p_shard.clone() if not self.params.is_cuda else self.p_shard,
                                        group=self.group)

    def shard_step(self):
        self.t += 1
        self.step_fn(self.p_shard, self.g_shard, self.s1, self.s2, self.absmax1, self.absmax2, self.t)

    def step(self):
        """reduce-scatter grads -> 8-bit step on the local shard -> all-gather params."""
        self.reduce_scatter()
        self.shard_step()
        self.all_gather()


def exchange_peer_tensors(tensors, group=None):
    """Map every rank's `tensors` into this process (CUDA IPC through torch's tensor sharing, the
    handles travelling over the process group).  Returns peers[r][k] = rank r's k-th tensor as a
    tensor of this process (own rank: the tensor itself).  Works across GPUs of a node (NVLink peer
    mappings) and between processes sharing one GPU."""
    from torch.multiprocessing.reductions import reduce_tensor
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = [reduce_tensor(t) for t in tensors]
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    peers = []
    for r in range(world):
        if r == rank:
            peers.append(list(tensors))
        else:
            peers.append([fn(*args) for fn, args in allh[r]])
    return peers


class ZeroFusedOptimizer8bit:
    """ZeRO-1 with the reduce-scatter, the 8-bit shard step and the all-gather fused into ONE kernel
    per rank over peer memory (q8_optim8bit_step_zero_fused): each rank reads
    its shard's gradients from every rank's buffer, steps the shard and writes the new values into
    every rank's parameter buffer, tile by tile; CTAs of the ranks meet at flag barriers in each
    rank's signal pad.  Buffers as Zero1Optimizer8bit (flat, padded to world*2048); the gradient
    of a shard is the rank-order binary32 sum / world (reading Z1).

    num_ctas: CTAs per rank (0 = one per SM).  Ranks that share one GPU (tests) must use at most
    SMs / world each so that every CTA of every rank can be resident.

    multicast: "auto" (default) allocates the gradient, parameter and signal buffers with torch's
    symmetric memory when every rank has its own GPU and the node supports NVLS multicast (NVSwitch):
    the peers' buffers come from its rendezvous instead of CUDA IPC, and the all-gather becomes one
    multimem.st per 16 bytes through the switch (the kernel's p_multicast).  "off" keeps IPC peer
    mappings and W peer stores; "on" requires multicast (raises otherwise)."""

    def __init__(self, n_params: int, kind: str = "adamw", grad_dtype=torch.bfloat16, device=None, group=None,
                 num_ctas: int = 0, multicast: str = "auto", **hparams):
        if kind not in ("adam", "adamw", "momentum"):
            raise ValueError("the fused ZeRO step takes adam / adamw / momentum")
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.kind = kind
        self.n = n_params
        self.n_pad = padded_numel(n_params, self.world)
        self.lo, self.hi = shard_range(self.n_pad, self.world, self.rank)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.num_ctas = num_ctas
        self.p_mc = None
        sig_bytes = B.zero_signal_bytes(self.world, num_ctas)
        handles = self._symmetric(dev, grad_dtype, sig_bytes, group) if multicast != "off" else None
        if handles is None and multicast == "on":
            raise RuntimeError("NVLS multicast is not available (needs one GPU per rank on an NVSwitch node)")
        if handles is None:
            self.params = torch.zeros(self.n_pad, dtype=torch.float32, device=dev)
            self.grads = torch.zeros(self.n_pad, dtype=grad_dtype, device=dev)
            self.signal = torch.zeros(sig_bytes, dtype=torch.uint8, device=dev)
        shard = self.hi - self.lo
        two = kind != "momentum"
        self.s1 = torch.zeros(shard, dtype=torch.uint8, device=dev)
        self.absmax1 = torch.zeros(shard // B.BLOCKSIZE, dtype=torch.float32, device=dev)
        self.s2 = torch.zeros(shard, dtype=torch.uint8, device=dev) if two else None
        self.absmax2 = torch.zeros(shard // B.BLOCKSIZE, dtype=torch.float32, device=dev) if two else None
        self.hp = B.hparams(**hparams)
        self.t = 0
        self.epoch = 0
        torch.cuda.synchronize(dev)
        if handles is not None:   # symmetric memory: peers' addresses and the multicast address
            hg, hp, hs = handles
            self._g, self._p, self._sig = list(hg.buffer_ptrs), list(hp.buffer_ptrs), list(hs.buffer_ptrs)
            self.p_mc = int(hp.multicast_ptr)
            self._peers = [[hg.get_buffer(r, (self.n_pad,), grad_dtype), hp.get_buffer(r, (self.n_pad,), torch.float32),
                            hs.get_buffer(r, (sig_bytes,), torch.uint8)] for r in range(self.world)]
            dist.barrier(group)
            return
        if self.world > 1:
            self._peers = exchange_peer_tensors([self.grads, self.params, self.signal], group)
            dist.barrier(group)
        else:
            self._peers = [[self.grads, self.params, self.signal]]
        self._g = [pt[0].data_ptr() for pt in self._peers]
        self._p = [pt[1].data_ptr() for pt in self._peers]
        self._sig = [pt[2].data_ptr() for pt in self._peers]

    def _symmetric(self, dev, grad_dtype, sig_bytes, group):
        """Allocate grads / params / signal pad in torch symmetric memory and rendezvous them, if the
        ranks have distinct GPUs and the node supports multicast; None otherwise."""
        if self.world < 2 or not dist.is_initialized() or dist.get_backend(group) != "nccl":
            return None
        try:
            import torch.distributed._symmetric_memory as symm
            if not symm._SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, dev.index):
                return None
            grp = group if group is not None else dist.group.WORLD
            bufs = [symm.empty(self.n_pad, dtype=grad_dtype, device=dev),
                    symm.empty(self.n_pad, dtype=torch.float32, device=dev),
                    symm.empty(sig_bytes, dtype=torch.uint8, device=dev)]
            for t in bufs:
                t.zero_()
            hs = [symm.rendezvous(t, grp) for t in bufs]
            if not int(getattr(hs[1], "multicast_ptr", 0) or 0):
                return None
        except Exception:  # noqa: BLE001  (no symmetric-memory backend / no multicast on this node)
            return None
        self.grads, self.params, self.signal = bufs
        return hs

    @property
    def p_shard(self) -> torch.Tensor:
        return self.params[self.lo:self.hi]

    def step(self):
        """One fused reduce-scatter + 8-bit step + all-gather (a single kernel launch)."""
        self.t += 1
        self.epoch += 1
        B.optim8bit_step_zero_fused(self.kind, self.world, self.rank, self._g, self._p, self._sig, self.s1, self.s2,
                                    self.absmax1, self.absmax2, self.n_pad, self.grads.dtype, step=self.t,
                                    epoch=self.epoch, num_ctas=self.num_ctas, hp=self.hp, p_multicast=self.p_mc)
