"""Build libspmat.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2406_08646_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libspmat.so")
SOURCES = ["comm.cu", "sf.cu", "coo.cu", "spmv.cu", "mult.cu", "halo.cu", "krylov.cu", "bsr.cu", "transpose.cu"]
HEADERS = [os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "halo_dev.cuh"), os.path.join(CSRC, "ptx.cuh"),
           os.path.join(ROOT, "include", "spmat.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def nccl_include() -> str:
    """NCCL headers for the types only (the library dlopen()s libnccl at run time)."""
    try:
        import nvidia.nccl  # type: ignore
        p = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(p, "nccl.h")):
            return p
    except Exception:
        pass
    return "/usr/include"


def _flags():
    return (["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
            + ARCH + ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_include()])


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s.replace(".cu", ".o"))
        if force or _stale(obj, [src] + HEADERS):
            cmd = [nvcc(), "-c", src, "-o", obj] + _flags()
            if verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for cmd, r in zip(jobs, results):
            if verbose or r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    objs = [os.path.join(OBJ, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + f".{os.getpid()}.tmp"
        cmd = [nvcc(), "-shared", "-o", tmp] + objs + ARCH + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
