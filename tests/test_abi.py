"""CPU-side checks of the C ABI (no GPU needed): libq8.so loads, exports every symbol that
include/q8.h declares, its host codebook matches the oracle bit for bit, and argument
validation fails synchronously with the documented status codes before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2110_02861_b200 as q8
from paper_2110_02861_b200 import _binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "q8.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(q8_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert set(syms) == set(B.EXPORTS), syms
    for s in syms:
        assert hasattr(B.lib, s), s
    out = os.popen(f"nm -D --defined-only {B.LIB_PATH}").read()
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {B.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


@pytest.mark.parametrize("signed", [True, False])
def test_host_codebook_matches_oracle(signed):
    a = q8.create_dynamic_codebook(signed).numpy()
    b = oracle.dynamic_codebook(signed)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _hp(**kw):
    d = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, bias_correction=True)
    d.update(kw)
    return B.hparams(**d)


FAKE = 1 << 20  # an aligned non-NULL address; validation fails before any dereference


@pytest.mark.parametrize("args,status", [
    (dict(n=-1), B.Q8_ERR_INVALID),
    (dict(blocksize=1024), B.Q8_ERR_UNSUPPORTED),
    (dict(gdt=7), B.Q8_ERR_INVALID),
    (dict(kind=9), B.Q8_ERR_INVALID),
    (dict(p=0), B.Q8_ERR_INVALID),
    (dict(p=FAKE + 4), B.Q8_ERR_INVALID),
    (dict(s1=FAKE + 1), B.Q8_ERR_INVALID),
    (dict(step=0), B.Q8_ERR_INVALID),
    (dict(hp=_hp(beta1=1.0)), B.Q8_ERR_INVALID),
    (dict(hp=_hp(eps=0.0)), B.Q8_ERR_INVALID),
    (dict(hp=_hp(lr=-1.0)), B.Q8_ERR_INVALID),
])
def test_step_validation(args, status):
    a = dict(kind=B.Q8_ADAM, p=FAKE, g=FAKE, gdt=B.Q8_BF16, s1=FAKE, s2=FAKE, a1=FAKE, a2=FAKE, n=4096,
             blocksize=2048, hp=_hp(), step=1)
    a.update(args)
    rc = B.lib.q8_optim8bit_step(a["kind"], a["p"], a["g"], a["gdt"], a["s1"], a["s2"], a["a1"], a["a2"], a["n"],
                                 a["blocksize"], ctypes.byref(a["hp"]), a["step"], None)
    assert rc == status
    assert B.lib.q8_last_error().decode() != ""


def test_zero_length_is_noop_without_device():
    rc = B.lib.q8_optim8bit_step(B.Q8_ADAM, 0, 0, B.Q8_F32, 0, 0, 0, 0, 0, 2048, ctypes.byref(_hp()), 1, None)
    assert rc == B.Q8_OK
    assert B.lib.q8_quantize_blockwise(0, 0, 0, 0, 0, 2048, None) == B.Q8_OK
    assert B.lib.q8_dequantize_blockwise(0, 0, 0, 0, 0, 2048, None) == B.Q8_OK


def test_codec_validation():
    assert B.lib.q8_quantize_blockwise(FAKE, FAKE, FAKE, FAKE, -5, 2048, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_quantize_blockwise(FAKE, FAKE + 8, FAKE, FAKE, 10, 2048, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_dequantize_blockwise(FAKE, FAKE, FAKE, FAKE, 10, 512, None) == B.Q8_ERR_UNSUPPORTED
    assert B.lib.q8_create_dynamic_codebook(1, None) == B.Q8_ERR_INVALID


def test_multi_validation():
    arr = (B.TensorDesc * 2)()
    arr[0] = B.TensorDesc(FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 100)
    arr[1] = B.TensorDesc(FAKE + 4, FAKE, FAKE, FAKE, FAKE, FAKE, 100)
    rc = B.lib.q8_optim8bit_step_multi(B.Q8_ADAM, B.Q8_F16, arr, 2, 2048, ctypes.byref(_hp()), 1, None)
    assert rc == B.Q8_ERR_INVALID and "tensor 1" in B.lib.q8_last_error().decode()
    assert B.lib.q8_optim8bit_step_multi(B.Q8_ADAM, B.Q8_F16, arr, -1, 2048, ctypes.byref(_hp()), 1,
                                         None) == B.Q8_ERR_INVALID


@pytest.mark.parametrize("signed", [True, False])
def test_host_linear_codebook_matches_oracle(signed):
    a = q8.create_linear_codebook(signed).numpy()
    b = oracle.linear_codebook(signed)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _lw(kind=B.Q8_LAMB, trust=0.001, ws=FAKE, ws_bytes=1 << 20, arr=None, count=1, hp=None):
    if arr is None:
        arr = (B.TensorDesc * 1)()
        arr[0] = B.TensorDesc(FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 5000)
    return B.lib.q8_optim8bit_step_layerwise(kind, B.Q8_BF16, arr, count, 2048, ctypes.byref(hp or _hp(eps=1e-6)),
                                             trust, 1, ws, ws_bytes, None)


def test_layerwise_scale_offset_matches_header():
    import re
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "q8.h")).read()
    m = re.search(r"#define Q8_LAYERWISE_SCALE_OFFSET (\d+)", hdr)
    assert m and int(m.group(1)) == B.Q8_LAYERWISE_SCALE_OFFSET == 4 * 384 + 16


def test_layerwise_workspace_bytes():
    arr = (B.TensorDesc * 3)()
    for i, n in enumerate((5000, 0, 2048)):
        arr[i] = B.TensorDesc(FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, n)
    # scales: 3 floats -> 16 B; partials: (3 + 0 + 1) blocks x 8 warp slots x 16 B; 384 LARS block
    # counters; 16 B grid barrier
    assert B.lib.q8_layerwise_workspace_bytes(arr, 3) == 16 + 4 * 128 + 4 * 384 + 16
    assert B.lib.q8_layerwise_workspace_bytes(arr, -1) == -1


def test_layerwise_validation():
    assert _lw(kind=B.Q8_ADAM) == B.Q8_ERR_INVALID
    assert _lw(kind=B.Q8_LARS, trust=0.0) == B.Q8_ERR_INVALID
    assert _lw(ws_bytes=16) == B.Q8_ERR_INVALID and "workspace too small" in B.lib.q8_last_error().decode()
    assert _lw(ws=FAKE + 8) == B.Q8_ERR_INVALID
    assert _lw(hp=_hp(eps=0.0)) == B.Q8_ERR_INVALID
    # layer-wise kinds are rejected by the element-wise entry points
    rc = B.lib.q8_optim8bit_step(B.Q8_LAMB, FAKE, FAKE, B.Q8_BF16, FAKE, FAKE, FAKE, FAKE, 4096, 2048,
                                 ctypes.byref(_hp()), 1, None)
    assert rc == B.Q8_ERR_INVALID and "layer-wise" in B.lib.q8_last_error().decode()


def test_quantile_validation_without_device():
    # argument checks happen before any device work (include/q8.h)
    assert B.lib.q8_estimate_quantiles(FAKE, 0, FAKE, None, FAKE, 1 << 20, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_estimate_quantiles(None, 10, FAKE, None, FAKE, 1 << 20, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_estimate_quantiles(FAKE + 4, 10, FAKE, None, FAKE, 1 << 20, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_create_quantile_codebook(None, None) == B.Q8_ERR_INVALID
    z = np.zeros(257, np.float32)
    out = np.zeros(256, np.float32)
    assert B.lib.q8_create_quantile_codebook(z.ctypes.data, out.ctypes.data) == B.Q8_ERR_INVALID


def test_host_quantile_codebook_matches_oracle():
    # host function of the library vs the oracle (independent implementations of Eq.5 / Q5)

    rng = np.random.default_rng(0)
    for q in (np.sort(rng.standard_normal(257)).astype(np.float32),
              np.sort(rng.exponential(size=257)).astype(np.float32) - np.float32(3.0),
              np.linspace(0, 1, 257).astype(np.float32)):
        lib_c = B.create_quantile_codebook(torch.from_numpy(q)).numpy()
        np.testing.assert_array_equal(lib_c.view(np.uint32), oracle.quantile_codebook(q).view(np.uint32))


def test_count_nonfinite_validation_without_device():
    assert B.lib.q8_count_nonfinite(FAKE, B.Q8_BF16, -1, FAKE, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_count_nonfinite(FAKE, B.Q8_BF16, 10, None, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_count_nonfinite(None, B.Q8_F32, 10, FAKE, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_count_nonfinite(FAKE + 2, B.Q8_F16, 10, FAKE, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_count_nonfinite(FAKE, 7, 10, FAKE, None) == B.Q8_ERR_INVALID


def test_binding_rejects_bad_tensors_before_the_c_call():
    # argument marshalling checks in the Python binding (no device needed): CPU tensors, sizes, dtypes
    p = torch.zeros(4096)
    g = torch.zeros(4096, dtype=torch.bfloat16)
    s = torch.zeros(4096, dtype=torch.uint8)
    a = torch.zeros(2)
    with pytest.raises(ValueError, match="CUDA"):
        q8.optim8bit_step("adamw", p, g, s, s.clone(), a, a.clone(), lr=1e-3, step=1)
    with pytest.raises(ValueError, match="size mismatch"):
        q8.optim8bit_step("adamw", p, g[:100], s, s.clone(), a, a.clone(), lr=1e-3, step=1)
    with pytest.raises(ValueError, match="unsupported gradient dtype"):
        q8.optim8bit_step("adam", p, g.to(torch.float64), s, s.clone(), a, a.clone(), lr=1e-3, step=1)
    with pytest.raises(ValueError):
        q8.count_nonfinite(torch.zeros(8, dtype=torch.int32))
    with pytest.raises(ValueError, match="257"):
        q8.create_quantile_codebook(torch.zeros(10))


def test_plan_validation_without_device():
    """q8_plan_*: argument validation happens before any CUDA call (kind, dtype, block size, tensor
    descriptors of both state widths, NULLs); the plan calls reject NULL plans."""
    arr = (B.TensorDesc * 2)()
    arr[0] = B.TensorDesc(FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 100)
    arr[1] = B.TensorDesc(FAKE, FAKE + 2, FAKE, FAKE, FAKE, FAKE, 100)   # misaligned gradient
    a32 = (B.TensorDesc32 * 1)()
    a32[0] = B.TensorDesc32(FAKE, FAKE, FAKE, 0, 100)                  # Adam needs r
    out = ctypes.c_void_p()
    create = B.lib.q8_plan_create
    assert create(B.Q8_ADAM, B.Q8_BF16, arr, 2, None, 0, 2048, ctypes.byref(out)) == B.Q8_ERR_INVALID
    assert "tensor 1" in B.lib.q8_last_error().decode()
    assert create(B.Q8_ADAM, B.Q8_BF16, arr, 1, a32, 1, 2048, ctypes.byref(out)) == B.Q8_ERR_INVALID
    assert "tensor 1" in B.lib.q8_last_error().decode()
    assert create(B.Q8_LAMB, B.Q8_BF16, arr, 1, None, 0, 2048, ctypes.byref(out)) == B.Q8_ERR_INVALID
    assert create(B.Q8_ADAM, 9, arr, 1, None, 0, 2048, ctypes.byref(out)) == B.Q8_ERR_INVALID
    assert create(B.Q8_ADAM, B.Q8_BF16, arr, 1, None, 0, 4096, ctypes.byref(out)) == B.Q8_ERR_UNSUPPORTED
    assert create(B.Q8_ADAM, B.Q8_BF16, None, 1, None, 0, 2048, ctypes.byref(out)) == B.Q8_ERR_INVALID
    assert create(B.Q8_ADAM, B.Q8_BF16, arr, 1, None, 0, 2048, None) == B.Q8_ERR_INVALID
    assert out.value is None
    g = (ctypes.c_void_p * 1)(FAKE)
    assert B.lib.q8_plan_set_grads(None, g, 1) == B.Q8_ERR_INVALID
    assert B.lib.q8_plan_step(None, ctypes.byref(_hp()), 1, None) == B.Q8_ERR_INVALID
    assert B.lib.q8_plan_step_device(None, ctypes.byref(_hp()), FAKE, None) == B.Q8_ERR_INVALID
    B.lib.q8_plan_destroy(None)


@pytest.mark.parametrize("kind,hpkey", [("adam", "adam"), ("adamw", "adamw"), ("lamb", "lamb")])
def test_host_step_scalars_follow_g8(kind, hpkey):
    """q8_step_scalars (host): the G8-G10 scalars each rounded once from binary64 -- checked here
    against numpy binary64 arithmetic for several steps (the device copy is compared with these on the
    GPU, tests/test_gpu_plan.py)."""
    h = dict(synth.HPARAMS[hpkey])
    h.pop("trust_coefficient", None)
    hp = q8.hparams(**h)
    for t in (1, 2, 10, 1000, 123456):
        s = q8.step_scalars(kind, hp, t).numpy()
        bc1 = 1.0 - np.power(np.float64(h["beta1"]), t)
        bc2 = 1.0 - np.power(np.float64(h["beta2"]), t)
        if kind == "lamb":
            step_size = np.sqrt(bc2) / bc1
        else:
            step_size = h["lr"] * np.sqrt(bc2) / bc1
        assert s[5] == np.float32(step_size)
        assert s[6] == np.float32(h["eps"] * np.sqrt(bc2))
        assert s[8] == np.float32(1.0 - h["lr"] * h["weight_decay"])
        assert s[3] == np.float32(1.0 - h["beta1"]) and s[4] == np.float32(1.0 - h["beta2"])
