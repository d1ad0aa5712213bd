"""CPU oracle for the block-wise dynamic 8-bit optimizer step -- TEST INFRASTRUCTURE ONLY.

Python (ctypes + numpy) shim over ``oracle/oracle.c``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import this package.  It never imports ``paper_2110_02861_b200`` and the
CUDA library never imports it.  See the header of ``oracle.c`` for the paper
passages each function follows and which pins (tests) hold it in place.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ADAM, ADAMW, MOMENTUM, LAMB, LARS = 0, 1, 2, 3, 4
KINDS = {"adam": ADAM, "adamw": ADAMW, "momentum": MOMENTUM, "lamb": LAMB, "lars": LARS}
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (plain gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


class _HParams(ctypes.Structure):
    _fields_ = [
        ("lr", ctypes.c_double),
        ("beta1", ctypes.c_double),
        ("beta2", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("weight_decay", ctypes.c_double),
        ("bias_correction", ctypes.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        l = ctypes.CDLL(build())
        f32p = ctypes.POINTER(ctypes.c_float)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        i64 = ctypes.c_int64
        l.oracle_dynamic_codebook.argtypes = [ctypes.c_int, f32p]
        l.oracle_linear_codebook.argtypes = [ctypes.c_int, f32p]
        l.oracle_nearest_code.argtypes = [f32p, ctypes.c_float]
        l.oracle_quantize_blockwise.argtypes = [f32p, f32p, i64, i64, f32p, u8p]
        l.oracle_dequantize_blockwise.argtypes = [f32p, u8p, f32p, i64, i64, f32p]
        l.oracle_optim32bit_step.argtypes = [ctypes.c_int, f32p, f32p, f32p, f32p, i64,
                                             ctypes.POINTER(_HParams), i64]
        l.oracle_optim8bit_step.argtypes = [ctypes.c_int, f32p, f32p, u8p, u8p, f32p, f32p, i64, i64,
                                            ctypes.POINTER(_HParams), i64, ctypes.c_int]
        l.oracle_optim32bit_layerwise_step.argtypes = [ctypes.c_int, f32p, f32p, f32p, f32p, i64,
                                                       ctypes.POINTER(_HParams), ctypes.c_double, i64, f32p, f32p]
        l.oracle_optim8bit_layerwise_step.argtypes = [ctypes.c_int, f32p, f32p, u8p, u8p, f32p, f32p, i64, i64,
                                                      ctypes.POINTER(_HParams), ctypes.c_double, i64, f32p, f32p]
        _lib = l
    return _lib


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _opt_ptr(a):
    """float32 pointer or NULL (the returned pointer keeps the array alive)."""
    return None if a is None else _ptr(a, ctypes.c_float)


def dynamic_codebook(signed: bool) -> np.ndarray:
    """256 ascending binary32 values of the (signed) dynamic tree / (unsigned) dynamic type."""
    out = np.zeros(256, np.float32)
    rc = lib().oracle_dynamic_codebook(1 if signed else 0, _ptr(out, ctypes.c_float))
    if rc != 0:
        raise RuntimeError("oracle codebook is not 256 distinct ascending values")
    return out


def linear_codebook(signed: bool) -> np.ndarray:
    """256 evenly spaced binary32 values over [-1, 1] (signed) / [0, 1] (T3 ablation baseline)."""
    out = np.zeros(256, np.float32)
    lib().oracle_linear_codebook(1 if signed else 0, _ptr(out, ctypes.c_float))
    return out


def nearest_code(Q: np.ndarray, y) -> np.ndarray:
    """Eq.3 argmin for each binary32 value in y (ties -> lower index)."""
    Q = _f32(Q)
    y = np.atleast_1d(_f32(y))
    qp = _ptr(Q, ctypes.c_float)
    f = lib().oracle_nearest_code
    return np.array([f(qp, ctypes.c_float(float(v))) for v in y], dtype=np.uint8)


def quantize_blockwise(Q: np.ndarray, x: np.ndarray, blocksize: int = 2048):
    """Eq.4: returns (absmax[ceil(n/B)] float32, codes[n] uint8)."""
    Q, x = _f32(Q), _f32(x)
    n = x.size
    absmax = np.zeros((n + blocksize - 1) // blocksize, np.float32)
    codes = np.zeros(n, np.uint8)
    rc = lib().oracle_quantize_blockwise(_ptr(Q, ctypes.c_float), _ptr(x, ctypes.c_float), n, blocksize,
                                         _ptr(absmax, ctypes.c_float), _ptr(codes, ctypes.c_uint8))
    if rc != 0:
        raise ValueError("invalid arguments")
    return absmax, codes


def dequantize_blockwise(Q: np.ndarray, codes: np.ndarray, absmax: np.ndarray, blocksize: int = 2048):
    Q, absmax = _f32(Q), _f32(absmax)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    out = np.zeros(codes.size, np.float32)
    rc = lib().oracle_dequantize_blockwise(_ptr(Q, ctypes.c_float), _ptr(codes, ctypes.c_uint8),
                                           _ptr(absmax, ctypes.c_float), codes.size, blocksize,
                                           _ptr(out, ctypes.c_float))
    if rc != 0:
        raise ValueError("invalid arguments")
    return out


def _hp(lr, beta1, beta2, eps, weight_decay, bias_correction) -> _HParams:
    return _HParams(float(lr), float(beta1), float(beta2), float(eps), float(weight_decay),
                    1 if bias_correction else 0)


def optim32bit_step(kind, p, g, m, r, *, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                    bias_correction=True, step=1):
    """In-place 32-bit step on float32 numpy arrays p, m, r (r ignored for momentum)."""
    kind = KINDS.get(kind, kind)
    for a in (p, m) + ((r,) if r is not None else ()):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    g = _f32(g)
    if r is None:
        r = np.zeros(1, np.float32)
    hp = _hp(lr, beta1, beta2, eps, weight_decay, bias_correction)
    rc = lib().oracle_optim32bit_step(kind, _ptr(p, ctypes.c_float), _ptr(g, ctypes.c_float),
                                      _ptr(m, ctypes.c_float), _ptr(r, ctypes.c_float), p.size,
                                      ctypes.byref(hp), int(step))
    if rc != 0:
        raise ValueError("invalid arguments")


def optim8bit_step(kind, p, g, s1, s2, absmax1, absmax2, *, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                   weight_decay=0.0, bias_correction=True, step=1, blocksize=2048, nthreads=1):
    """In-place 8-bit step.  p float32, g float32 (16-bit grads widened by the caller),
    s1/s2 uint8 codes, absmax1/absmax2 float32 per block.  s2/absmax2 unused for momentum."""
    kind = KINDS.get(kind, kind)
    for a, dt in ((p, np.float32), (s1, np.uint8), (absmax1, np.float32)):
        assert a.dtype == dt and a.flags.c_contiguous
    g = _f32(g)
    if s2 is None:
        s2 = np.zeros(1, np.uint8)
        absmax2 = np.zeros(1, np.float32)
    hp = _hp(lr, beta1, beta2, eps, weight_decay, bias_correction)
    rc = lib().oracle_optim8bit_step(kind, _ptr(p, ctypes.c_float), _ptr(g, ctypes.c_float),
                                     _ptr(s1, ctypes.c_uint8), _ptr(s2, ctypes.c_uint8),
                                     _ptr(absmax1, ctypes.c_float), _ptr(absmax2, ctypes.c_float),
                                     p.size, blocksize, ctypes.byref(hp), int(step), int(nthreads))
    if rc != 0:
        raise ValueError("invalid arguments")


def _forced(scale):
    return None if scale is None else np.array([scale], np.float32)


def optim32bit_layerwise_step(kind, p, g, m, r, *, lr, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.0,
                              bias_correction=True, step=1, trust_coefficient=0.001, forced_scale=None):
    """In-place 32-bit LAMB / LARS step over ONE tensor (readings L1-L4 in oracle.c).  p, m, r
    float32 (r LAMB only).  Returns the fp32 per-tensor scale RN(lr*trust ratio).  forced_scale:
    use this fp32 scale instead of the one from the norms (teacher forcing, reading L3)."""
    kind = KINDS.get(kind, kind)
    for a in (p, m) + ((r,) if kind == LAMB else ()):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    g = _f32(g)
    if r is None:
        r = np.zeros(1, np.float32)
    hp = _hp(lr, beta1, beta2, eps, weight_decay, bias_correction)
    out = np.zeros(1, np.float32)
    rc = lib().oracle_optim32bit_layerwise_step(kind, _ptr(p, ctypes.c_float), _ptr(g, ctypes.c_float),
                                                _ptr(m, ctypes.c_float), _ptr(r, ctypes.c_float), p.size,
                                                ctypes.byref(hp), float(trust_coefficient), int(step),
                                                _ptr(out, ctypes.c_float), _opt_ptr(_forced(forced_scale)))
    if rc != 0:
        raise ValueError("invalid arguments")
    return out[0]


def optim8bit_layerwise_step(kind, p, g, s1, s2, absmax1, absmax2, *, lr, beta1=0.9, beta2=0.999, eps=1e-6,
                             weight_decay=0.0, bias_correction=True, step=1, trust_coefficient=0.001,
                             blocksize=2048, forced_scale=None):
    """In-place 8-bit LAMB / LARS step over ONE tensor (s2/absmax2 LAMB only).  Returns the
    fp32 per-tensor scale.  forced_scale: as optim32bit_layerwise_step."""
    kind = KINDS.get(kind, kind)
    for a, dt in ((p, np.float32), (s1, np.uint8), (absmax1, np.float32)):
        assert a.dtype == dt and a.flags.c_contiguous
    g = _f32(g)
    if s2 is None:
        s2 = np.zeros(1, np.uint8)
        absmax2 = np.zeros(1, np.float32)
    hp = _hp(lr, beta1, beta2, eps, weight_decay, bias_correction)
    out = np.zeros(1, np.float32)
    rc = lib().oracle_optim8bit_layerwise_step(kind, _ptr(p, ctypes.c_float), _ptr(g, ctypes.c_float),
                                               _ptr(s1, ctypes.c_uint8), _ptr(s2, ctypes.c_uint8),
                                               _ptr(absmax1, ctypes.c_float), _ptr(absmax2, ctypes.c_float),
                                               p.size, blocksize, ctypes.byref(hp), float(trust_coefficient),
                                               int(step), _ptr(out, ctypes.c_float), _opt_ptr(_forced(forced_scale)))
    if rc != 0:
        raise ValueError("invalid arguments")
    return out[0]


def _quantile_lib():
    l = lib()
    if not getattr(l, "_quantiles_bound", False):
        f32p = ctypes.POINTER(ctypes.c_float)
        l.oracle_exact_quantiles.argtypes = [f32p, ctypes.c_int64, f32p]
        l.oracle_sram_quantiles.argtypes = [f32p, ctypes.c_int64, ctypes.c_int64, f32p]
        l.oracle_quantile_codebook.argtypes = [f32p, f32p]
        l._quantiles_bound = True
    return l


def exact_quantiles(x: np.ndarray) -> np.ndarray:
    """Sample quantiles Q(j/257), j = 0..256, of the whole tensor (App G; readings Q1, Q2)."""
    x = _f32(x).ravel()
    out = np.zeros(257, np.float32)
    if _quantile_lib().oracle_exact_quantiles(_ptr(x, ctypes.c_float), x.size, _ptr(out, ctypes.c_float)) != 0:
        raise ValueError("invalid arguments")
    return out


def sram_quantiles(x: np.ndarray, subset: int = 4096) -> np.ndarray:
    """SRAM-Quantiles (App G; readings Q1-Q4): per-chunk sample quantiles, averaged."""
    x = _f32(x).ravel()
    out = np.zeros(257, np.float32)
    if _quantile_lib().oracle_sram_quantiles(_ptr(x, ctypes.c_float), x.size, int(subset),
                                             _ptr(out, ctypes.c_float)) != 0:
        raise ValueError("invalid arguments")
    return out


def quantile_codebook(quantiles: np.ndarray) -> np.ndarray:
    """Quantile data type from 257 quantiles (Eq.5, reading Q5): 256 values in [-1, 1]."""
    q = _f32(quantiles)
    assert q.size == 257
    out = np.zeros(256, np.float32)
    if _quantile_lib().oracle_quantile_codebook(_ptr(q, ctypes.c_float), _ptr(out, ctypes.c_float)) != 0:
        raise ValueError("all Eq.5 midpoints are zero")
    return out
