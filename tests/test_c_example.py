"""The boundary is a plain C ABI: examples/c_abi_step.c (no Python, no torch) compiles against
include/q8.h with gcc as C11 and links libq8.so (CPU check); on a GPU it runs 8-bit AdamW steps and
checks the t = 1 closed form |dw| = lr*|g|/(|g|+eps) after the decoupled decay (GPU check)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2110_02861_b200")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    exe = str(tmp_path / "c_abi_step")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "c_abi_step.c"), "-L", PKG, "-lq8", "-I", f"{CUDA}/include",
           "-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{PKG}", "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = _build(tmp_path)
    for n in ("1", "2047", "1000003"):
        r = subprocess.run([exe, n], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "c_abi_step ok" in r.stdout, r.stdout + r.stderr
