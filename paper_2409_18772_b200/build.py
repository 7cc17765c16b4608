"""Build liblrqmm.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2409_18772_b200.build [--force]

Each .cu is compiled separately (in parallel) with
`-gencode arch=compute_100a,code=sm_100a -lineinfo -O3` (no fast-math: the
scale lambda needs IEEE division, reading #4) and linked against the
CUDA runtime and the venv's NCCL (rpath baked in, so the .so loads on the GPU
box that has the same image).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "liblrqmm.so")
SOURCES = ["quantize.cu", "skinny.cu", "skinny_tc.cu", "smallsolve2.cu", "gemm_i8.cu", "comm.cu", "lrqmm_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    import nvidia.nccl  # the venv's NCCL wheel (same one torch uses)

    return os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else list(nvidia.nccl.__path__)[0]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl = _nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include")]
    extra = os.environ.get("LRQMM_EXTRA_NVCC", "").split()
    flags = extra + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             "--expt-relaxed-constexpr"] + ARCH + inc
    # every header of csrc/ is a dependency of every object (solvers.cuh was missing from a fixed list)
    hdrs = sorted(os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))) + [os.path.join(ROOT, "include", f) for f in ("lrqmm.h", "lrqmm_debug.h")]
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([nvcc(), "-c", s, "-o", o] + flags)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for out in ex.map(run, jobs):
            if verbose and out:
                print(out)
    if force or _stale(LIB, objs):
        link = [nvcc(), "-shared", "-o", LIB] + objs + ARCH + [
            "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-lcudart",
            "-Xlinker", "-rpath," + os.path.join(nccl, "lib"), "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        run(link)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
