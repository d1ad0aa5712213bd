"""Build libq8.so in-tree: nvcc for sm_100a only (no PTX JIT fallback), cudart static.

The step kernels are instantiated per gradient dtype (step_inst.cu compiled three times with
-DQ8_GDT=0/1/2); the objects compile in parallel and link into one shared library."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libq8.so")
OBJDIR = os.environ.get("Q8_OBJDIR", "/tmp/q8_build")
UNITS = [("q8_api.cu", []), ("codebook_host.cpp", []),
         ("step_inst.cu", ["-DQ8_GDT=0"]), ("step_inst.cu", ["-DQ8_GDT=1"]), ("step_inst.cu", ["-DQ8_GDT=2"])]
HEADERS = ["q8_kernels.cuh", "q8_codec.cuh", "q8_step32_kernel.cuh", "q8_step_kernel.cuh", "q8_layerwise.cuh", "q8_quantiles.cuh", "q8_quant_kernel.cuh", "q8_launch.h", os.path.join("..", "..", "include", "q8.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17",
    # IEEE fp32 everywhere: bit-exact parity with the oracle depends on it (G9)
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false", "-fmad=false",
    "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v,-warn-spills",
] + os.environ.get("Q8_EXTRA_NVCC_FLAGS", "").split()


def _obj(src, defs):
    tag = "".join(d.split("=")[-1] for d in defs)
    return os.path.join(OBJDIR, os.path.splitext(src)[0] + (f"_g{tag}" if tag else "") + ".o")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f, _ in UNITS] + [os.path.join(CSRC, h) for h in HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, defs):
    out = _obj(src, defs)
    cmd = [NVCC, *NVCC_FLAGS, *defs, "-c", "-o", out, os.path.join(CSRC, src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, defs, r


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(len(UNITS), os.cpu_count() or 1)) as ex:
        for src, defs, r in ex.map(lambda u: _compile(*u), UNITS):
            logs.append(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src} {defs}")
    lib = os.environ.get("Q8_LIB_OUT", LIB)
    tmp = lib + f".tmp{os.getpid()}"
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp] + [_obj(s, d) for s, d in UNITS]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed for libq8.so")
    if verbose:
        sys.stderr.write("".join(logs))
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
