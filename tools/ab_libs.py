"""A/B of library builds on the flat cfg4 step (development tool): each .so given on the command line is
loaded with ctypes and q8_optim8bit_step (stable ABI) is device-timed on the same buffers, interleaved."""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402


class HP(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double), ("bias_correction", ctypes.c_int32)]


libs = []
for path in sys.argv[1:]:
    lib = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.q8_optim8bit_step.argtypes = [i32, vp, vp, i32, vp, vp, vp, vp, i64, i32, ctypes.POINTER(HP), i64, vp]
    libs.append((path.split("/")[-1], lib))
n = synth.workload_numel("cfg4_gpt2_xl")
dev = "cuda"
p = synth.params(n, device=dev)
gs = [synth.grads(n, step=t, dtype="bfloat16", device=dev) for t in (1, 2)]
s1, a1 = synth.zero_state(n, device=dev)
s2, a2 = synth.zero_state(n, device=dev)
h = synth.HPARAMS["adamw"]
hp = HP(h["lr"], h["beta1"], h["beta2"], h["eps"], h["weight_decay"], 1)
t = [0]


def step(lib):
    t[0] += 1
    r = lib.q8_optim8bit_step(1, p.data_ptr(), gs[t[0] % 2].data_ptr(), 2, s1.data_ptr(), s2.data_ptr(), a1.data_ptr(),
                              a2.data_ptr(), n, 2048, ctypes.byref(hp), t[0], torch.cuda.current_stream().cuda_stream)
    assert r == 0


for _ in range(10):
    step(libs[0][1])
torch.cuda.synchronize()
res = {name: [] for name, _ in libs}
iters = int(__import__("os").environ.get("AB_ITERS", "20"))
for rep in range(6):
    for name, lib in libs:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for a, b in ev:
            a.record()
            step(lib)
            b.record()
        torch.cuda.synchronize()
        res[name].append(statistics.mean(a.elapsed_time(b) for a, b in ev))
print({k: [round(x, 4) for x in v] for k, v in res.items()})
print({k: round(statistics.median(v), 4) for k, v in res.items()})
