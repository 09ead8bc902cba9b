"""Build libgemm_f16.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgemm_f16.so")
ROOT = os.path.dirname(PKG)

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "gemm_f16.h")])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build_variant(out: str, defines=()) -> str:
    """A/B build of the same sources with extra -D flags into `out` (tools/ab_libs.py,
    tools/ab_power.py); never the product library."""
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], os.path.join(CSRC, "gemm_api.cu"), "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    return out


FASTBIND_DIR = os.path.join(PKG, "_fastbind")
FASTBIND_SO = os.path.join(FASTBIND_DIR, "gemm_f16_fastbind.so")
FASTBIND_SRC = os.path.join(CSRC, "fastbind.cpp")


def build_fastbind(force: bool = False) -> str:
    """The torch-tensor fast path of the Python binding (csrc/fastbind.cpp: argument marshalling
    only), compiled in-tree with torch.utils.cpp_extension.  Optional: the ctypes path is used
    when it is absent."""
    if not force and os.path.exists(FASTBIND_SO) and os.path.getmtime(FASTBIND_SO) >= os.path.getmtime(FASTBIND_SRC):
        return FASTBIND_SO
    from torch.utils import cpp_extension
    os.makedirs(FASTBIND_DIR, exist_ok=True)
    cpp_extension.load(name="gemm_f16_fastbind", sources=[FASTBIND_SRC], build_directory=FASTBIND_DIR,
                       extra_cflags=["-O2"], with_cuda=True, verbose=False)
    return FASTBIND_SO


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, os.path.join(CSRC, "gemm_api.cu"), "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    with open(os.path.join(PKG, "csrc", "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    if verbose:
        print(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
