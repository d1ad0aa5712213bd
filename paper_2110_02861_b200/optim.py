"""torch.optim-style 8-bit optimizers over the fused sm_100a step (the paper's "two-line
change", P:7 / P:28: swap the optimizer class).

Each parameter keeps its optimizer state as 8-bit codes plus one fp32 absmax per 2048-element
block (S3.1): ``s1``/``absmax1`` for the first state (signed dynamic tree type),
``s2``/``absmax2`` for Adam's second state (unsigned dynamic type).  Tensors marked with
``_q8_optim_bits = 32`` (the StableEmbedding weight, S3.3 P:124) or in a param group with
``optim_bits=32`` keep fp32 states ``m``/``r`` instead (``q8_optim32bit_step_multi``).  A step groups all
parameters that have gradients by gradient dtype and calls ``q8_optim8bit_step_multi`` once
per group (one kernel launch per <= 384 tensors).  Parameters must be fp32, contiguous and
16-byte aligned on a CUDA device; there is no CPU path.
"""
from __future__ import annotations

from collections import defaultdict

import torch

from . import _binding as B


_TWO_STATES = ("adam", "adamw", "lamb")


class _Version:
    """Modification counter shared by an optimizer's state containers."""
    __slots__ = ("v",)

    def __init__(self):
        self.v = 0

    def __getstate__(self):
        return self.v

    def __setstate__(self, v):
        self.v = v


def _tracked(base):
    """A dict / defaultdict subclass whose every structural change bumps `self._ver.v`: a cached
    plan holds raw pointers to the state tensors, so replacing or resetting any state (opt.state.clear(),
    opt.state[p] = {}, st["s1"] = new tensor) must invalidate it (the version check is O(1) per step)."""
    class Tracked(base):
        def __setitem__(self, k, v):
            self._ver.v += 1
            super().__setitem__(k, v)

        def __delitem__(self, k):
            self._ver.v += 1
            super().__delitem__(k)

        def clear(self):
            self._ver.v += 1
            super().clear()

        def pop(self, *a):
            self._ver.v += 1
            return super().pop(*a)

        def popitem(self):
            self._ver.v += 1
            return super().popitem()

        def update(self, *a, **k):
            self._ver.v += 1
            super().update(*a, **k)

        def setdefault(self, k, d=None):
            if k not in self:
                self._ver.v += 1
            return super().setdefault(k, d)
    return Tracked


_TrackedDict = _tracked(dict)
_TrackedDefaultDict = _tracked(defaultdict)


class _ParamState(_TrackedDict):
    def __init__(self, ver, *a, **k):
        self._ver = ver
        super().__init__(*a, **k)

    def __reduce__(self):
        return (_ParamState, (self._ver, dict(self)))


class _StateFactory:
    def __init__(self, ver):
        self.ver = ver

    def __call__(self):
        return _ParamState(self.ver)


class _States(_TrackedDefaultDict):
    def __init__(self, ver, items=()):
        self._ver = ver
        super().__init__(_StateFactory(ver))
        for k, v in dict(items).items():
            dict.__setitem__(self, k, _ParamState(ver, v))

    def __reduce__(self):
        return (_States, (self._ver, dict(self)))


class _GroupPlan:
    """A cached plan (q8_plan) over the parameters of one param group that have gradients of one
    dtype and one step count: their 8-bit- and 32-bit-state tensors are stepped by the same
    launch(es).  The step counter is shared by the plan's tensors: a host int (`t`) or, in
    capturable mode, a device int64 tensor (`step_t`) that the kernel advances."""

    def __init__(self, opt, group, params, gdt, capturable):
        st = opt.state
        p8 = [p for p in params if "s1" in st[p]]
        p32 = [p for p in params if "s1" not in st[p]]
        e8 = [(p, p.grad, st[p]["s1"], st[p].get("s2"), st[p]["absmax1"], st[p].get("absmax2")) for p in p8]
        e32 = [(p, p.grad, st[p]["m"], st[p].get("r")) for p in p32]
        self.plan = B.Plan(opt.kind, e8, e32)
        self.params = p8 + p32
        self.states = [st[p] for p in self.params]   # the state dicts this plan steps
        self.gdt = gdt
        pos = {id(p): i for i, p in enumerate(group["params"])}
        self.idx = [pos[id(p)] for p in self.params]       # positions in group["params"]
        self.pptrs = [p.data_ptr() for p in self.params]
        self.t = None
        self.step_t = None
        s0 = st[self.params[0]]["step"]
        if capturable:
            self.step_t = (s0.detach().to(device=self.plan.device, dtype=torch.int64).reshape(1).clone()
                           if torch.is_tensor(s0) else
                           torch.full((1,), int(s0), dtype=torch.int64, device=self.plan.device))
            for p in self.params:
                dict.__setitem__(st[p], "step", self.step_t)   # not a structural change of the state
        else:
            self.t = int(s0)


class _Optimizer8bit(torch.optim.Optimizer):
    kind = "adam"

    def __init__(self, params, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0, bias_correction=True,
                 capturable=False):
        """capturable: keep each plan's step counter on the device (state["step"] is a shared int64 CUDA
        tensor advanced by the kernel), so that step() can be captured in a CUDA graph and replayed
        with no host work (q8_plan_step_device)."""
        if lr < 0 or eps <= 0 or not (0 <= betas[0] < 1) or not (0 <= betas[1] < 1) or weight_decay < 0:
            raise ValueError("invalid hyper-parameters")
        super().__init__(params, dict(lr=lr, betas=tuple(betas), eps=eps, weight_decay=weight_decay,
                                      bias_correction=bias_correction, capturable=capturable))
        self._ver = _Version()
        self.state = _States(self._ver, self.state)
        self._lists = {}
        self._plans = {}   # id(group) -> (state version, mask of params with grads, [_GroupPlan])

    @staticmethod
    def _bits(p: torch.Tensor, group) -> int:
        # per-tensor override (StableEmbedding sets _q8_optim_bits = 32, S3.3 P:124) or group key
        return int(getattr(p, "_q8_optim_bits", None) or group.get("optim_bits", 8))

    def _state_for(self, p: torch.Tensor, bits: int):
        st = self.state[p]
        if not st:
            if p.dtype != torch.float32 or not p.is_cuda:
                raise TypeError("8-bit optimizers update fp32 CUDA parameters")
            n = p.numel()
            st["step"] = 0
            if bits == 32:
                st["m"] = torch.zeros(n, dtype=torch.float32, device=p.device)
                if self.kind in _TWO_STATES:
                    st["r"] = torch.zeros(n, dtype=torch.float32, device=p.device)
            else:
                nb = B.nblocks(n)
                st["s1"] = torch.zeros(n, dtype=torch.uint8, device=p.device)
                st["absmax1"] = torch.zeros(nb, dtype=torch.float32, device=p.device)
                if self.kind in _TWO_STATES:
                    st["s2"] = torch.zeros(n, dtype=torch.uint8, device=p.device)
                    st["absmax2"] = torch.zeros(nb, dtype=torch.float32, device=p.device)
        return st

    def _tensor_list(self, group, gdt, entries):
        """The multi-tensor descriptor array for these entries (layer-wise optimizers), cached per
        (group, dtype, parameter and state storage): a parameter whose .data is re-pointed, or a
        state that was reset or replaced, gets a new key; gradients are refreshed in place."""
        key = (id(group), gdt, tuple((e[0].data_ptr(), e[2].data_ptr(), e[4].data_ptr(),
                                      e[3].data_ptr() if e[3] is not None else 0,
                                      e[5].data_ptr() if e[5] is not None else 0) for e in entries))
        tl = self._lists.get(key)
        if tl is None:
            tl = B.TensorList(entries, self.kind)
            if len(self._lists) > 64:
                self._lists.clear()
            self._lists[key] = tl
        else:
            tl.update_grads([e[1] for e in entries])
        return tl

    def load_state_dict(self, state_dict):
        # torch casts floating-point-param state to the param dtype; codes must stay uint8
        super().load_state_dict(state_dict)
        self.state = _States(self._ver, self.state)
        self._ver.v += 1
        for st in self.state.values():
            for k in ("m", "r"):
                if k in st:
                    st[k] = st[k].to(torch.float32).contiguous()
            for k in ("s1", "s2"):
                if k in st:
                    st[k] = st[k].to(torch.uint8).contiguous()
            for k in ("absmax1", "absmax2"):
                if k in st:
                    st[k] = st[k].to(torch.float32).contiguous()
            if "step" in st and not torch.is_tensor(st["step"]):
                st["step"] = int(st["step"])
        self._lists.clear()
        self._plans.clear()

    def state_dict(self):
        self._sync_steps()
        return super().state_dict()

    def _sync_steps(self):
        """Host-stepped plans keep one counter per plan; write it back into every tensor's state."""
        for _, _, gps in self._plans.values():
            for gp in gps:
                if gp.t is not None:
                    for st in gp.states:  # (a state dict dropped from opt.state since is left alone)
                        dict.__setitem__(st, "step", gp.t)

    def _fast(self, group):
        """The cached plans of a group with this step's gradients, if nothing they depend on changed:
        the same parameters have gradients (of the plan's dtype, contiguous), parameter storage is
        unchanged and no state was replaced (version counter).  None otherwise."""
        c = self._plans.get(id(group))
        if c is None or c[0] != self._ver.v:
            return None
        gall = [p.grad for p in group["params"]]
        if [g is None for g in gall] != c[1]:
            return None
        out = []
        for gp in c[2]:
            grads = [gall[i] for i in gp.idx]
            dt = gp.gdt
            if not all(g.dtype is dt and g.is_contiguous() for g in grads):
                return None
            if [p.data_ptr() for p in gp.params] != gp.pptrs:
                return None
            out.append((gp, grads))
        return out

    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        for group in self.param_groups:
            b1, b2 = group["betas"]
            hp = B.hparams(group["lr"], b1, b2, group["eps"], group["weight_decay"], group["bias_correction"])
            plans = self._fast(group)
            if plans is None:
                plans = self._build_plans(group)
            for gp, grads in plans:
                gp.plan.set_grad_ptrs([g.data_ptr() for g in grads], grads)
                if gp.step_t is not None:
                    gp.plan.step_device(hp, gp.step_t)
                else:
                    gp.t += 1
                    gp.plan.step(hp, gp.t)
        return loss

    def _build_plans(self, group):
        """(Re)build the plans of a group: every parameter with a gradient, bucketed by gradient dtype
        and current step count (the tensors of one plan share the counter)."""
        self._sync_steps()
        self._plans.pop(id(group), None)
        buckets = {}
        grads = {}
        for p in group["params"]:
            if p.grad is None:
                continue
            if p.grad.is_sparse:
                raise TypeError("sparse gradients are not supported")
            if not p.grad.is_contiguous():
                raise ValueError("8-bit optimizers need contiguous gradients")
            st = self._state_for(p, self._bits(p, group))
            s = st["step"]
            key = (p.grad.dtype, int(s) if not torch.is_tensor(s) else int(s.item()))
            buckets.setdefault(key, []).append(p)
        gps = []
        for (gdt, _), params in buckets.items():
            gps.append(_GroupPlan(self, group, params, gdt, group.get("capturable", False)))
        mask = [p.grad is None for p in group["params"]]
        self._plans[id(group)] = (self._ver.v, mask, gps)
        return [(gp, [p.grad for p in gp.params]) for gp in gps]


class Adam8bit(_Optimizer8bit):
    """Adam (Eq.2) with 8-bit block-wise dynamic states; L2 weight decay."""
    kind = "adam"


class AdamW8bit(_Optimizer8bit):
    """AdamW: Adam with decoupled weight decay (Loshchilov & Hutter, cited P:134)."""
    kind = "adamw"

    def __init__(self, params, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=1e-2, bias_correction=True,
                 capturable=False):
        super().__init__(params, lr, betas, eps, weight_decay, bias_correction, capturable)


class Momentum8bit(_Optimizer8bit):
    """SGD with momentum, Eq.1: m = beta*m + g, w -= lr*m (no dampening)."""
    kind = "momentum"

    def __init__(self, params, lr=0.1, momentum=0.9, weight_decay=0.0, capturable=False):
        super().__init__(params, lr, (momentum, 0.0), 1e-8, weight_decay, False, capturable)


class _LayerwiseOptimizer8bit(_Optimizer8bit):
    """Layer-wise (trust-ratio) optimizers: every parameter tensor is one layer with its own
    trust ratio (q8_optim8bit_step_layerwise: norms pass, per-tensor scale, fused step).  The
    per-tensor scales RN(lr * ratio) of the last step are kept in ``state[p]["trust_scale"]``
    (a 0-d float32 CUDA tensor)."""
    trust_coefficient = 0.001

    def __init__(self, params, lr, betas, eps, weight_decay, bias_correction):
        super().__init__(params, lr, betas, eps, weight_decay, bias_correction)
        self._workspace = None

    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        for group in self.param_groups:
            buckets = {}
            for p in group["params"]:
                if p.grad is None:
                    continue
                if p.grad.is_sparse:
                    raise TypeError("sparse gradients are not supported")
                if self._bits(p, group) != 8:
                    raise NotImplementedError("layer-wise 8-bit optimizers keep 8-bit states only")
                st = self._state_for(p, 8)
                st["step"] += 1
                g = p.grad if p.grad.is_contiguous() else p.grad.contiguous()
                buckets.setdefault((g.dtype, st["step"]), []).append(
                    (p, g, st["s1"], st.get("s2"), st["absmax1"], st.get("absmax2")))
            b1, b2 = group["betas"]
            hp = B.hparams(group["lr"], b1, b2, group["eps"], group["weight_decay"], group["bias_correction"])
            eta = group.get("trust_coefficient", self.trust_coefficient)
            for (gdt, step), entries in buckets.items():
                tl = self._tensor_list(group, gdt, entries)
                need = B.layerwise_workspace_bytes(tl)
                if self._workspace is None or self._workspace.numel() < need:
                    self._workspace = torch.zeros(need, dtype=torch.uint8, device=tl.device)  # zero-filled (q8.h)
                scales = B.optim8bit_step_layerwise(self.kind, tl, lr=group["lr"], step=step, hp=hp,
                                                    trust_coefficient=eta, workspace=self._workspace).clone()
                for i, e in enumerate(entries):
                    self.state[e[0]]["trust_scale"] = scales[i]
        return loss


class LAMB8bit(_LayerwiseOptimizer8bit):
    """LAMB (You et al. 2020, Alg. 2; T5 P:366) with 8-bit block-wise dynamic states: Adam
    moments, u = m_hat/(sqrt(r_hat)+eps) + wd*w, w -= lr * ||w||/||u|| * u per tensor."""
    kind = "lamb"

    def __init__(self, params, lr=1e-3, betas=(0.9, 0.999), eps=1e-6, weight_decay=0.01, bias_correction=True):
        super().__init__(params, lr, betas, eps, weight_decay, bias_correction)


class LARS8bit(_LayerwiseOptimizer8bit):
    """LARS (You et al. 2017, Alg. 1; T5 P:367) with an 8-bit block-wise momentum state:
    v = momentum*v + lr * eta*||w||/(||g|| + wd*||w||) * (g + wd*w), w -= v per tensor."""
    kind = "lars"

    def __init__(self, params, lr=0.1, momentum=0.9, weight_decay=5e-4, trust_coefficient=0.001):
        if trust_coefficient <= 0:
            raise ValueError("trust_coefficient must be > 0")
        super().__init__(params, lr, (momentum, 0.0), 1e-8, weight_decay, False)
        for group in self.param_groups:
            group.setdefault("trust_coefficient", trust_coefficient)


def state_bytes(n_params: int, kind: str = "adam", blocksize: int = B.BLOCKSIZE) -> int:
    """Optimizer-state bytes of the 8-bit optimizer: 1 B per element per state plus one fp32
    absmax per block per state (8 GB -> 2 GB for a 1B-parameter Adam)."""
    states = 2 if kind in _TWO_STATES else 1
    return states * (n_params + 4 * B.nblocks(n_params, blocksize))
