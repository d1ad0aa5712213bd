"""Thin ctypes binding over libq8.so (include/q8.h).  Argument marshalling only: every step
of the hot path runs in the CUDA kernels of csrc/.  There is no CPU fallback; if the
library cannot be loaded, importing this module raises."""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# Q8_LIB_PATH: development A/B override of the library file (tools/probe_step.py)
LIB_PATH = os.environ.get("Q8_LIB_PATH") or os.path.join(_HERE, "libq8.so")

Q8_OK, Q8_ERR_INVALID, Q8_ERR_UNSUPPORTED, Q8_ERR_CUDA = 0, -1, -2, -3
Q8_F32, Q8_F16, Q8_BF16 = 0, 1, 2
Q8_ADAM, Q8_ADAMW, Q8_MOMENTUM, Q8_LAMB, Q8_LARS = 0, 1, 2, 3, 4
MAX_TENSORS_PER_LAUNCH = 384
BLOCKSIZE = 2048
Q8_LAYERWISE_SCALE_OFFSET = 1552  # include/q8.h: the layer-wise scales' byte offset in the workspace

KINDS = {"adam": Q8_ADAM, "adamw": Q8_ADAMW, "momentum": Q8_MOMENTUM, "lamb": Q8_LAMB, "lars": Q8_LARS}
GDTYPES = {torch.float32: Q8_F32, torch.float16: Q8_F16, torch.bfloat16: Q8_BF16}

EXPORTS = ("q8_create_dynamic_codebook", "q8_create_linear_codebook", "q8_quantize_blockwise",
           "q8_quantize_blockwise_dynamic", "q8_dequantize_blockwise", "q8_quantize_tensorwise",
           "q8_dequantize_tensorwise",
           "q8_optim8bit_step", "q8_optim8bit_step_multi", "q8_optim32bit_step_multi",
           "q8_optim8bit_step_layerwise", "q8_layerwise_workspace_bytes", "q8_optim8bit_step_zero_fused",
           "q8_zero_signal_bytes", "q8_estimate_quantiles", "q8_quantiles_workspace_bytes",
           "q8_create_quantile_codebook", "q8_count_nonfinite", "q8_plan_create", "q8_plan_set_grads",
           "q8_plan_step", "q8_plan_step_device", "q8_step_scalars", "q8_step_scalars_device",
           "q8_plan_destroy", "q8_last_error", "q8_version")


class Q8Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"q8 status {status}: {msg}")
        self.status = status


class HParams(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double), ("bias_correction", ctypes.c_int32)]


class TensorDesc32(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p), ("g", ctypes.c_void_p), ("m", ctypes.c_void_p), ("r", ctypes.c_void_p),
                ("n", ctypes.c_int64)]


class TensorDesc(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p), ("g", ctypes.c_void_p), ("s1", ctypes.c_void_p), ("s2", ctypes.c_void_p),
                ("absmax1", ctypes.c_void_p), ("absmax2", ctypes.c_void_p), ("n", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.q8_create_dynamic_codebook.argtypes = [i32, vp]
    lib.q8_create_linear_codebook.argtypes = [i32, vp]
    lib.q8_quantize_tensorwise.argtypes = [vp, vp, vp, vp, i64, vp]
    lib.q8_dequantize_tensorwise.argtypes = [vp, vp, vp, vp, i64, vp]
    lib.q8_quantize_blockwise.argtypes = [vp, vp, vp, vp, i64, i32, vp]
    lib.q8_quantize_blockwise_dynamic.argtypes = [i32, vp, vp, vp, i64, i32, vp]
    lib.q8_dequantize_blockwise.argtypes = [vp, vp, vp, vp, i64, i32, vp]
    lib.q8_optim8bit_step.argtypes = [i32, vp, vp, i32, vp, vp, vp, vp, i64, i32, ctypes.POINTER(HParams), i64, vp]
    lib.q8_optim8bit_step_multi.argtypes = [i32, i32, ctypes.POINTER(TensorDesc), i32, i32,
                                            ctypes.POINTER(HParams), i64, vp]
    lib.q8_optim32bit_step_multi.argtypes = [i32, i32, ctypes.POINTER(TensorDesc32), i32, ctypes.POINTER(HParams),
                                             i64, vp]
    lib.q8_optim8bit_step_layerwise.argtypes = [i32, i32, ctypes.POINTER(TensorDesc), i32, i32,
                                                ctypes.POINTER(HParams), ctypes.c_double, i64, vp, i64, vp]
    lib.q8_layerwise_workspace_bytes.argtypes = [ctypes.POINTER(TensorDesc), i32]
    lib.q8_optim8bit_step_zero_fused.argtypes = [i32, i32, i32, i32, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                                 ctypes.POINTER(vp), vp, vp, vp, vp, vp, i64, i32,
                                                 ctypes.POINTER(HParams), i64, ctypes.c_uint32, i32, vp]
    lib.q8_zero_signal_bytes.argtypes = [i32, i32]
    lib.q8_estimate_quantiles.argtypes = [vp, i64, vp, vp, vp, i64, vp]
    lib.q8_quantiles_workspace_bytes.argtypes = [i64]
    lib.q8_create_quantile_codebook.argtypes = [vp, vp]
    lib.q8_count_nonfinite.argtypes = [vp, i32, i64, vp, vp]
    lib.q8_plan_create.argtypes = [i32, i32, ctypes.POINTER(TensorDesc), i32, ctypes.POINTER(TensorDesc32), i32, i32,
                                   ctypes.POINTER(vp)]
    lib.q8_plan_set_grads.argtypes = [vp, ctypes.POINTER(vp), i32]
    lib.q8_plan_step.argtypes = [vp, ctypes.POINTER(HParams), i64, vp]
    lib.q8_plan_step_device.argtypes = [vp, ctypes.POINTER(HParams), vp, vp]
    lib.q8_plan_destroy.argtypes = [vp]
    lib.q8_step_scalars.argtypes = [i32, ctypes.POINTER(HParams), i64, vp]
    lib.q8_step_scalars_device.argtypes = [i32, ctypes.POINTER(HParams), vp, i64, vp, vp]
    for f in EXPORTS[:-3]:
        getattr(lib, f).restype = ctypes.c_int
    lib.q8_plan_destroy.restype = None
    lib.q8_layerwise_workspace_bytes.restype = i64
    lib.q8_zero_signal_bytes.restype = i64
    lib.q8_quantiles_workspace_bytes.restype = i64
    lib.q8_last_error.restype = ctypes.c_char_p
    lib.q8_version.restype = ctypes.c_char_p
    return lib


lib = _load()


def _check(status: int):
    if status != Q8_OK:
        raise Q8Error(status, lib.q8_last_error().decode())


def _stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _dev_ptr(t: torch.Tensor | None, dtype=None, name="tensor", device=None) -> int | None:
    """Device address of a contiguous CUDA tensor; `device` (if given) is the device of the call:
    every buffer of one call must live on it (the C ABI launches on the current device)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, but this call runs on {device}")
    return t.data_ptr()


def _on(device):
    """Make `device` current for one C call: the library takes its tables, SM count and launch
    device from the current CUDA device, and the stream handle is that device's current stream."""
    if torch.device(device).type != "cuda":
        raise ValueError(f"the 8-bit kernels take CUDA tensors (got a tensor on {device})")
    return torch.cuda.device(device)


def version() -> str:
    return lib.q8_version().decode()


def nblocks(n: int, blocksize: int = BLOCKSIZE) -> int:
    return (n + blocksize - 1) // blocksize


def create_dynamic_codebook(signed: bool) -> torch.Tensor:
    """Host call: the 256 ascending fp32 values of the (un)signed dynamic data type."""
    out = torch.empty(256, dtype=torch.float32)
    _check(lib.q8_create_dynamic_codebook(1 if signed else 0, out.data_ptr()))
    return out


def create_linear_codebook(signed: bool) -> torch.Tensor:
    """Host call: the 256 evenly spaced fp32 values of the linear data type (ablation baseline)."""
    out = torch.empty(256, dtype=torch.float32)
    _check(lib.q8_create_linear_codebook(1 if signed else 0, out.data_ptr()))
    return out


def quantize_tensorwise(code: torch.Tensor, x: torch.Tensor, absmax: torch.Tensor | None = None,
                        codes: torch.Tensor | None = None):
    """Eq.3: one absmax for the whole tensor, then the nearest code of x/N."""
    n, dev = x.numel(), x.device
    if absmax is None:
        absmax = torch.empty(1, dtype=torch.float32, device=dev)
    if codes is None:
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
    if codes.numel() != n or absmax.numel() < 1 or code.numel() != 256:
        raise ValueError("size mismatch")
    with _on(dev):
        _check(lib.q8_quantize_tensorwise(_dev_ptr(code, torch.float32, "code", dev), _dev_ptr(x, torch.float32, "x"),
                                          _dev_ptr(absmax, torch.float32, "absmax", dev),
                                          _dev_ptr(codes, torch.uint8, "codes", dev), n, _stream(dev)))
    return absmax, codes


def dequantize_tensorwise(code: torch.Tensor, codes: torch.Tensor, absmax: torch.Tensor,
                          out: torch.Tensor | None = None):
    n, dev = codes.numel(), codes.device
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=dev)
    if out.numel() != n or absmax.numel() < 1 or code.numel() != 256:
        raise ValueError("size mismatch")
    with _on(dev):
        _check(lib.q8_dequantize_tensorwise(_dev_ptr(code, torch.float32, "code", dev),
                                            _dev_ptr(codes, torch.uint8, "codes"),
                                            _dev_ptr(absmax, torch.float32, "absmax", dev),
                                            _dev_ptr(out, torch.float32, "out", dev), n, _stream(dev)))
    return out


def quantize_blockwise(code: torch.Tensor, x: torch.Tensor, absmax: torch.Tensor | None = None,
                       codes: torch.Tensor | None = None, blocksize: int = BLOCKSIZE):
    n, dev = x.numel(), x.device
    if absmax is None:
        absmax = torch.empty(nblocks(n, blocksize), dtype=torch.float32, device=dev)
    if codes is None:
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
    if codes.numel() != n or absmax.numel() < nblocks(n, blocksize) or code.numel() != 256:
        raise ValueError("size mismatch")
    with _on(dev):
        _check(lib.q8_quantize_blockwise(_dev_ptr(code, torch.float32, "code", dev), _dev_ptr(x, torch.float32, "x"),
                                         _dev_ptr(absmax, torch.float32, "absmax", dev),
                                         _dev_ptr(codes, torch.uint8, "codes", dev), n, blocksize, _stream(dev)))
    return absmax, codes


def quantize_blockwise_dynamic(signed: bool, x: torch.Tensor, absmax: torch.Tensor | None = None,
                               codes: torch.Tensor | None = None, blocksize: int = BLOCKSIZE):
    """Eq.4 with the library's built-in dynamic data type (the step kernel's search path)."""
    n, dev = x.numel(), x.device
    if absmax is None:
        absmax = torch.empty(nblocks(n, blocksize), dtype=torch.float32, device=dev)
    if codes is None:
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
    if codes.numel() != n or absmax.numel() < nblocks(n, blocksize):
        raise ValueError("size mismatch")
    with _on(dev):
        _check(lib.q8_quantize_blockwise_dynamic(1 if signed else 0, _dev_ptr(x, torch.float32, "x"),
                                                 _dev_ptr(absmax, torch.float32, "absmax", dev),
                                                 _dev_ptr(codes, torch.uint8, "codes", dev), n, blocksize,
                                                 _stream(dev)))
    return absmax, codes


def dequantize_blockwise(code: torch.Tensor, codes: torch.Tensor, absmax: torch.Tensor,
                         out: torch.Tensor | None = None, blocksize: int = BLOCKSIZE):
    n, dev = codes.numel(), codes.device
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=dev)
    if out.numel() != n or absmax.numel() < nblocks(n, blocksize) or code.numel() != 256:
        raise ValueError("size mismatch")
    with _on(dev):
        _check(lib.q8_dequantize_blockwise(_dev_ptr(code, torch.float32, "code", dev),
                                           _dev_ptr(codes, torch.uint8, "codes"),
                                           _dev_ptr(absmax, torch.float32, "absmax", dev),
                                           _dev_ptr(out, torch.float32, "out", dev), n, blocksize, _stream(dev)))
    return out


def hparams(lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, bias_correction=True) -> HParams:
    return HParams(float(lr), float(beta1), float(beta2), float(eps), float(weight_decay),
                   1 if bias_correction else 0)


def _check_state_sizes(i, n, kind, g, s1, s2, a1, a2):
    """Sizes the C ABI cannot see: every buffer of a tensor holds n elements (absmax: one per
    2048-block), and the second state exists exactly for the two-state kinds."""
    two = kind in (Q8_ADAM, Q8_ADAMW, Q8_LAMB)
    nb = nblocks(n)
    if g.numel() != n or s1.numel() != n or a1.numel() < nb:
        raise ValueError(f"tensor {i}: size mismatch (g, s1 need {n} elements, absmax1 {nb})")
    if two and (s2 is None or a2 is None or s2.numel() != n or a2.numel() < nb):
        raise ValueError(f"tensor {i}: size mismatch (s2 needs {n} elements, absmax2 {nb})")


def optim8bit_step(kind, p, g, s1, s2, absmax1, absmax2, *, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                   weight_decay=0.0, bias_correction=True, step=1, blocksize=BLOCKSIZE, hp: HParams | None = None):
    """One fused 8-bit step on a single flat tensor (in place)."""
    kind = KINDS.get(kind, kind)
    n, dev = p.numel(), p.device
    _check_state_sizes(0, n, kind, g, s1, s2, absmax1, absmax2)
    if g.dtype not in GDTYPES:
        raise ValueError(f"unsupported gradient dtype {g.dtype}")
    if hp is None:
        hp = hparams(lr, beta1, beta2, eps, weight_decay, bias_correction)
    with _on(dev):
        _check(lib.q8_optim8bit_step(kind, _dev_ptr(p, torch.float32, "p"), _dev_ptr(g, None, "g", dev),
                                     GDTYPES[g.dtype], _dev_ptr(s1, torch.uint8, "s1", dev),
                                     _dev_ptr(s2, torch.uint8, "s2", dev),
                                     _dev_ptr(absmax1, torch.float32, "absmax1", dev),
                                     _dev_ptr(absmax2, torch.float32, "absmax2", dev), n, blocksize, ctypes.byref(hp),
                                     int(step), _stream(dev)))


class TensorList:
    """A prepared (cached) host descriptor array for optim8bit_step_multi."""

    def __init__(self, entries, kind=None):
        """entries: iterable of (p, g, s1, s2_or_None, absmax1, absmax2_or_None) CUDA tensors, all on
        one device.  kind (optional): checks that the second state is present for Adam/AdamW/LAMB."""
        entries = list(entries)
        self.arr = (TensorDesc * max(1, len(entries)))()
        self.count = len(entries)
        self.gdtype = None
        self.keep = entries  # keep tensors alive
        self.device = entries[0][0].device if entries else None
        kind = KINDS.get(kind, kind)
        dev = self.device
        for i, (p, g, s1, s2, a1, a2) in enumerate(entries):
            n = p.numel()
            if kind is not None:
                _check_state_sizes(i, n, kind, g, s1, s2, a1, a2)
            elif g.numel() != n or s1.numel() != n or a1.numel() < nblocks(n) or \
                    (s2 is not None and (s2.numel() != n or a2 is None or a2.numel() < nblocks(n))):
                raise ValueError(f"tensor {i}: size mismatch")
            if g.dtype not in GDTYPES:
                raise ValueError(f"tensor {i}: unsupported gradient dtype {g.dtype}")
            gd = GDTYPES[g.dtype]
            if self.gdtype is None:
                self.gdtype = gd
            elif gd != self.gdtype:
                raise ValueError("all gradients of one multi-tensor launch must share a dtype")
            self.arr[i] = TensorDesc(_dev_ptr(p, torch.float32, f"tensor {i} p", dev), _dev_ptr(g, None, f"tensor {i} g", dev),
                                     _dev_ptr(s1, torch.uint8, f"tensor {i} s1", dev),
                                     _dev_ptr(s2, torch.uint8, f"tensor {i} s2", dev),
                                     _dev_ptr(a1, torch.float32, f"tensor {i} absmax1", dev),
                                     _dev_ptr(a2, torch.float32, f"tensor {i} absmax2", dev), n)

    def update_grads(self, grads):
        """Re-point the descriptors at this step's gradients (same count, sizes, dtype and device as
        before); everything else (parameters, states) is unchanged, so no re-validation."""
        if len(grads) != self.count:
            raise ValueError("gradient count changed")
        arr, gd, dev = self.arr, self.gdtype, self.device
        for i, g in enumerate(grads):
            if g.device != dev or GDTYPES.get(g.dtype) != gd or g.numel() != arr[i].n:
                raise ValueError(f"tensor {i}: gradient device/size/dtype changed")
            arr[i].g = g.data_ptr()
        self.grads = grads  # keep this step's gradients alive until the next refresh


def optim8bit_step_multi(kind, tensors, *, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                         bias_correction=True, step=1, blocksize=BLOCKSIZE, hp: HParams | None = None):
    """One fused 8-bit step over many tensors (one launch per <= 384 tensors)."""
    kind = KINDS.get(kind, kind)
    tl = tensors if isinstance(tensors, TensorList) else TensorList(tensors, kind)
    if tl.count == 0:
        return
    if hp is None:
        hp = hparams(lr, beta1, beta2, eps, weight_decay, bias_correction)
    with _on(tl.device):
        _check(lib.q8_optim8bit_step_multi(kind, tl.gdtype, tl.arr, tl.count, blocksize, ctypes.byref(hp), int(step),
                                           _stream(tl.device)))


def optim32bit_step_multi(kind, tensors, *, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                          bias_correction=True, step=1, hp: HParams | None = None):
    """The same fp32 update with 32-bit states (m, r fp32 tensors): entries (p, g, m, r_or_None)."""
    kind = KINDS.get(kind, kind)
    entries = list(tensors)
    if not entries:
        return
    dev = entries[0][0].device
    arr = (TensorDesc32 * len(entries))()
    gd = None
    for i, (p, g, m, r) in enumerate(entries):
        n = p.numel()
        if g.numel() != n or m.numel() != n or (r is not None and r.numel() != n) or \
                (kind != Q8_MOMENTUM and r is None):
            raise ValueError(f"tensor {i}: size mismatch")
        if g.dtype not in GDTYPES:
            raise ValueError(f"tensor {i}: unsupported gradient dtype {g.dtype}")
        if gd is None:
            gd = GDTYPES[g.dtype]
        elif GDTYPES[g.dtype] != gd:
            raise ValueError("all gradients of one launch must share a dtype")
        arr[i] = TensorDesc32(_dev_ptr(p, torch.float32, "p", dev), _dev_ptr(g, None, "g", dev),
                              _dev_ptr(m, torch.float32, "m", dev), _dev_ptr(r, torch.float32, "r", dev), n)
    if hp is None:
        hp = hparams(lr, beta1, beta2, eps, weight_decay, bias_correction)
    with _on(dev):
        _check(lib.q8_optim32bit_step_multi(kind, gd, arr, len(entries), ctypes.byref(hp), int(step), _stream(dev)))


def layerwise_workspace_bytes(tensors) -> int:
    tl = tensors if isinstance(tensors, TensorList) else TensorList(tensors)
    nb = lib.q8_layerwise_workspace_bytes(tl.arr, tl.count)
    if nb < 0:
        raise ValueError("invalid tensor list")
    return nb


def optim8bit_step_layerwise(kind, tensors, *, lr, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.0,
                             bias_correction=True, step=1, trust_coefficient=0.001, blocksize=BLOCKSIZE,
                             workspace: torch.Tensor | None = None, hp: HParams | None = None) -> torch.Tensor:
    """One 8-bit LAMB / LARS step over many tensors (each tensor is one layer: its own trust
    ratio).  entries as optim8bit_step_multi (s2/absmax2 None for LARS).  workspace: a uint8 device
    tensor of at least layerwise_workspace_bytes() bytes whose first Q8_LAYERWISE_SCALE_OFFSET bytes
    are zero before its first use (torch.zeros; every call leaves them zero); None or too small:
    a zero-filled one is allocated.  Returns the float32 per-tensor scales RN(lr * ratio) (a view
    into the workspace, valid until its next use)."""
    kind = KINDS.get(kind, kind)
    tl = tensors if isinstance(tensors, TensorList) else TensorList(tensors, kind)
    if tl.count == 0:
        return torch.empty(0, dtype=torch.float32)
    need = lib.q8_layerwise_workspace_bytes(tl.arr, tl.count)
    if need < 0:
        raise ValueError("invalid tensor list")
    if workspace is None or workspace.numel() < need:
        workspace = torch.zeros(need, dtype=torch.uint8, device=tl.device)  # zero-filled (q8.h)
    if hp is None:
        hp = hparams(lr, beta1, beta2, eps, weight_decay, bias_correction)
    with _on(tl.device):
        _check(lib.q8_optim8bit_step_layerwise(kind, tl.gdtype, tl.arr, tl.count, blocksize, ctypes.byref(hp),
                                               float(trust_coefficient), int(step),
                                               _dev_ptr(workspace, torch.uint8, "workspace", tl.device),
                                               workspace.numel(), _stream(tl.device)))
    return workspace[Q8_LAYERWISE_SCALE_OFFSET:Q8_LAYERWISE_SCALE_OFFSET + 4 * tl.count].view(torch.float32)


def zero_signal_bytes(world: int, num_ctas: int = 0) -> int:
    nb = lib.q8_zero_signal_bytes(int(world), int(num_ctas))
    if nb < 0:
        raise ValueError("invalid world / num_ctas")
    return nb


def optim8bit_step_zero_fused(kind, world, rank, g_ptrs, p_ptrs, sig_ptrs, s1, s2, absmax1, absmax2, n_pad, g_dtype,
                              *, step, epoch, num_ctas=0, stream=None, hp: HParams, p_multicast=None):
    """Fused ZeRO-1 step over peer memory (q8_optim8bit_step_zero_fused): g_ptrs / p_ptrs /
    sig_ptrs are per-rank device addresses (ints) of the gradient, parameter and signal buffers;
    p_multicast (int or None) the NVLS multicast address of the parameter buffers."""
    kind = KINDS.get(kind, kind)
    dev = s1.device
    arr = ctypes.c_void_p * world
    with _on(dev):
        _check(lib.q8_optim8bit_step_zero_fused(kind, GDTYPES[g_dtype], world, rank, arr(*g_ptrs), arr(*p_ptrs),
                                                arr(*sig_ptrs), p_multicast, _dev_ptr(s1, torch.uint8, "s1"),
                                                _dev_ptr(s2, torch.uint8, "s2", dev),
                                                _dev_ptr(absmax1, torch.float32, "absmax1", dev),
                                                _dev_ptr(absmax2, torch.float32, "absmax2", dev), int(n_pad),
                                                BLOCKSIZE, ctypes.byref(hp), int(step), int(epoch), int(num_ctas),
                                                stream if stream is not None else _stream(dev)))


def quantiles_workspace_bytes(n: int, device=None) -> int:
    with _on(device if device is not None else torch.cuda.current_device()):
        nb = lib.q8_quantiles_workspace_bytes(int(n))
    if nb < 0:
        raise Q8Error(Q8_ERR_INVALID, lib.q8_last_error().decode() or "invalid n")
    return nb


def estimate_quantiles(x: torch.Tensor, *, with_codebook: bool = False, workspace: torch.Tensor | None = None,
                       quantiles: torch.Tensor | None = None, code: torch.Tensor | None = None):
    """SRAM-Quantiles (App G): the 257 quantiles Q(j/257) of x (fp32, on the GPU).  With
    with_codebook, also the Eq.5 quantile data type (256 fp32 in [-1, 1], on the GPU), usable
    as the `code` table of quantize_blockwise.  Returns quantiles or (quantiles, code)."""
    n, dev = x.numel(), x.device
    need = quantiles_workspace_bytes(n, dev)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    if quantiles is None:
        quantiles = torch.empty(257, dtype=torch.float32, device=dev)
    if with_codebook and code is None:
        code = torch.empty(256, dtype=torch.float32, device=dev)
    if quantiles.numel() != 257 or (code is not None and code.numel() != 256):
        raise ValueError("size mismatch")
    with _on(dev):
        _check(lib.q8_estimate_quantiles(_dev_ptr(x, torch.float32, "x"), n,
                                         _dev_ptr(quantiles, torch.float32, "quantiles", dev),
                                         _dev_ptr(code, torch.float32, "code", dev) if with_codebook else None,
                                         _dev_ptr(workspace, torch.uint8, "workspace", dev), workspace.numel(),
                                         _stream(dev)))
    return (quantiles, code) if with_codebook else quantiles


def create_quantile_codebook(quantiles) -> torch.Tensor:
    """Host call: the Eq.5 quantile data type from 257 quantiles (reading Q5)."""
    q = torch.as_tensor(quantiles, dtype=torch.float32).detach().cpu().contiguous()
    if q.numel() != 257:
        raise ValueError("need 257 quantiles")
    out = torch.empty(256, dtype=torch.float32)
    _check(lib.q8_create_quantile_codebook(q.data_ptr(), out.data_ptr()))
    return out


def count_nonfinite(g: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Number of NaN / inf elements of a gradient tensor, as a 1-element int64 CUDA tensor (no host
    sync): the AMP-style guard before an 8-bit step (non-finite gradients are out of contract)."""
    if g.dtype not in GDTYPES:
        raise ValueError(f"unsupported gradient dtype {g.dtype}")
    dev = g.device
    if out is None:
        out = torch.empty(1, dtype=torch.int64, device=dev)
    with _on(dev):
        _check(lib.q8_count_nonfinite(_dev_ptr(g, None, "g"), GDTYPES[g.dtype], g.numel(),
                                      _dev_ptr(out, torch.int64, "out", dev), _stream(dev)))
    return out


def step_scalars(kind, hp: HParams, step: int) -> torch.Tensor:
    """Host diagnostics: the ten fp32 scalars of one update (q8_step_scalars)."""
    out = torch.empty(10, dtype=torch.float32)
    _check(lib.q8_step_scalars(KINDS.get(kind, kind), ctypes.byref(hp), int(step), out.data_ptr()))
    return out


def step_scalars_device(kind, hp: HParams, steps: torch.Tensor) -> torch.Tensor:
    """The same ten scalars for every int64 step of `steps` (CUDA), computed on the device by the code
    the capturable plan step runs (q8_step_scalars_device); returns [n, 10] float32 on the device."""
    dev = steps.device
    out = torch.empty(steps.numel(), 10, dtype=torch.float32, device=dev)
    with _on(dev):
        _check(lib.q8_step_scalars_device(KINDS.get(kind, kind), ctypes.byref(hp), _dev_ptr(steps, torch.int64, "steps"),
                                          steps.numel(), _dev_ptr(out, torch.float32, "out", dev), _stream(dev)))
    return out


class Plan:
    """A prepared multi-tensor step (q8_plan_*): the descriptors of every tensor are validated and
    kept by the library once; a step is one call (one launch per 384 tensors).  entries8: (p, g, s1,
    s2_or_None, absmax1, absmax2_or_None); entries32: (p, g, m, r_or_None) -- tensors whose states
    stay fp32 (the Stable Embedding, S3.3 P:124), stepped in the SAME launch.  Tensor k of the plan is
    entries8[k], then entries32."""

    def __init__(self, kind, entries8=(), entries32=()):
        self.kind = KINDS.get(kind, kind)
        entries8, entries32 = list(entries8), list(entries32)
        alle = entries8 + entries32
        if not alle:
            raise ValueError("a plan needs at least one tensor")
        self.device = alle[0][0].device
        self.count = len(alle)
        tl = TensorList(entries8, self.kind) if entries8 else None
        gd = tl.gdtype if tl else None
        arr32 = (TensorDesc32 * max(1, len(entries32)))()
        dev = self.device
        for i, (p, g, m, r) in enumerate(entries32):
            n = p.numel()
            if g.numel() != n or m.numel() != n or (r is not None and r.numel() != n) or \
                    (self.kind != Q8_MOMENTUM and r is None):
                raise ValueError(f"32-bit tensor {i}: size mismatch")
            if GDTYPES.get(g.dtype) is None or (gd is not None and GDTYPES[g.dtype] != gd):
                raise ValueError("all gradients of one plan must share a dtype")
            gd = GDTYPES[g.dtype]
            arr32[i] = TensorDesc32(_dev_ptr(p, torch.float32, "p", dev), _dev_ptr(g, None, "g", dev),
                                    _dev_ptr(m, torch.float32, "m", dev), _dev_ptr(r, torch.float32, "r", dev), n)
        self.gdtype = gd
        self._gdt_torch = {v: k for k, v in GDTYPES.items()}[gd]
        self._numel = [e[0].numel() for e in alle]
        self.keep = alle  # the library holds raw pointers: keep every tensor alive
        h = ctypes.c_void_p()
        with _on(dev):
            _check(lib.q8_plan_create(self.kind, gd, tl.arr if tl else None, len(entries8), arr32, len(entries32),
                                      BLOCKSIZE, ctypes.byref(h)))
        self._h = h
        self._gptr = (ctypes.c_void_p * self.count)()

    def set_grads(self, grads):
        """Re-point the gradients (same count, sizes, dtype and device as the plan's)."""
        if len(grads) != self.count:
            raise ValueError("gradient count changed")
        gdt, dev = self._gdt_torch, self.device
        for i, (g, n) in enumerate(zip(grads, self._numel)):
            if g.dtype != gdt or g.device != dev or g.numel() != n or not g.is_contiguous():
                raise ValueError(f"tensor {i}: gradient dtype/device/size changed or not contiguous")
        self.set_grad_ptrs([g.data_ptr() for g in grads], grads)

    def set_grad_ptrs(self, ptrs, keep=None):
        """Re-point the gradients by address (the caller has checked dtype, size, device and
        contiguity -- the optimizer's fast path); `keep` is held until the next refresh."""
        self._gptr[:] = ptrs
        _check(lib.q8_plan_set_grads(self._h, self._gptr, self.count))
        self.grads = keep

    def step(self, hp: HParams, step: int):
        with _on(self.device):
            _check(lib.q8_plan_step(self._h, ctypes.byref(hp), int(step), _stream(self.device)))

    def step_device(self, hp: HParams, step_t: torch.Tensor):
        """Capturable step: t - 1 is read from step_t (int64 CUDA tensor of one element) on the device
        and t is stored back when the step completes; no host value changes between calls, so the
        call can be captured in a CUDA graph."""
        with _on(self.device):
            _check(lib.q8_plan_step_device(self._h, ctypes.byref(hp), _dev_ptr(step_t, torch.int64, "step",
                                                                                 self.device),
                                           _stream(self.device)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:
            lib.q8_plan_destroy(h)
            self._h = None
