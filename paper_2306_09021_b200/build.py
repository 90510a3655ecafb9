"""Build libpbng.so in-tree with nvcc for sm_100a (B200).  No torch extension machinery: the library is a
plain C-ABI shared object loaded with ctypes (paper_2306_09021_b200/pbng.py).

pbng_kernels.cu is compiled once per (dtype, model) -- each object holds that pair's sweep and energy /
residual instantiations -- plus once for the dispatchers and model-independent kernels, in parallel,
then linked with the host library (static cudart)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
HOST = os.path.join(CSRC, "pbng_host.cpp")
KERNELS = os.path.join(CSRC, "pbng_kernels.cu")
SOURCES = [HOST, KERNELS]
HEADERS = [os.path.join(CSRC, "pbng_internal.h"), os.path.join(ROOT, "include", "pbng.h")]
LIB = os.path.join(HERE, "libpbng.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
         "-I", CSRC, "--expt-relaxed-constexpr", "--diag-suppress=177"]
# (PBNG_TU_R, PBNG_TU_MODEL) of the per-instantiation objects; None = the dispatcher object
UNITS = [None] + [(r, m) for r in ("float", "double") for m in ("MODEL_NH", "MODEL_FCR", "MODEL_SNH")]


def stale(out: str = LIB) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


CACHE = os.path.join(ROOT, "build", "obj")  # objects of the last default build (tuning variants reuse them)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB, jobs: int = 0,
          only=None) -> str:
    """Compile the library; `defines` (e.g. ["PBNG_SWEEP_MINB=12"]) build tuning variants into `out`.
    only = [(R, MODEL), ...]: apply `defines` to those kernel objects only and reuse the cached default
    objects for the rest (a variant for one workload in a fraction of the time)."""
    if not force and not defines and out == LIB and not stale():
        return LIB
    tag = f"{os.path.basename(out)}.{os.getpid()}"
    objdir = os.path.join(os.path.dirname(out), f".obj_{tag}")
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(CACHE, exist_ok=True)
    extra = [*(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines]]
    default = not defines

    def compile_unit(unit):
        name = "kernels_common.o" if unit is None else f"kernels_{unit[0]}_{unit[1]}.o"
        cached = os.path.join(CACHE, name)
        if only is not None and unit not in only and not stale(cached):
            return cached
        if unit is None:
            src, o, udef = KERNELS, os.path.join(objdir, name), []
        else:
            r, m = unit
            src, o = KERNELS, os.path.join(objdir, name)
            udef = [f"-DPBNG_TU_R={r}", f"-DPBNG_TU_MODEL={m}"]
        use = extra if (only is None or unit in only) else []
        subprocess.check_call([NVCC, *ARCH, *FLAGS, *use, *udef, "-c", "-o", o, src])
        if default or (only is not None and unit not in only):
            import shutil
            shutil.copyfile(o, cached)
        return o

    def compile_host():
        o = os.path.join(objdir, "host.o")
        subprocess.check_call([NVCC, *ARCH, *FLAGS, *extra, "-c", "-o", o, HOST])
        return o

    jobs = jobs or max(1, min(len(UNITS) + 1, os.cpu_count() or 1))
    try:
        with ThreadPoolExecutor(jobs) as ex:
            futs = [ex.submit(compile_unit, u) for u in UNITS] + [ex.submit(compile_host)]
            objs = [f.result() for f in futs]
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
        os.replace(tmp, out)
    finally:
        for f in os.listdir(objdir):
            os.remove(os.path.join(objdir, f))
        os.rmdir(objdir)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
