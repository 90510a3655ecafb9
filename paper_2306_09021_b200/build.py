"""Build libpbng.so in-tree with nvcc for sm_100a (B200).  No torch extension machinery: the library is a
plain C-ABI shared object loaded with ctypes (paper_2306_09021_b200/pbng.py)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, "pbng_host.cpp"), os.path.join(CSRC, "pbng_kernels.cu")]
HEADERS = [os.path.join(CSRC, "pbng_internal.h"), os.path.join(ROOT, "include", "pbng.h")]
LIB = os.path.join(HERE, "libpbng.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Compile the library; `defines` (e.g. ["PBNG_SWEEP_MINB=12"]) build tuning variants into `out`."""
    if not force and not defines and out == LIB and not stale():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines],
           "-o", tmp, *SOURCES]
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
