"""Build libtrime_gpu.so in-tree for sm_100a (explicit nvcc, no JIT cache).

``python -m paper_2309_13824_b200.build`` or ``build()`` from Python.  The
library is rebuilt only when a source is newer than it (or force=True).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libtrime_gpu.so")
SOURCES = ["tm_api.cu", "tm_cells.cu", "tm_cells_t.cu", "tm_distmesh.cu", "tm_control.cu", "tm_setup.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=true",                   # decision arithmetic uses __d*_rn intrinsics (never contracted)
    "-Xcompiler", "-fPIC,-ffp-contract=off",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    srcs = [os.path.join(PKG, "csrc", s) for s in SOURCES]
    deps = srcs + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "trime_gpu.h")]
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    tmp = out + f".tmp{os.getpid()}"
    # one nvcc per translation unit, in parallel, then one shared-library link
    from concurrent.futures import ThreadPoolExecutor
    objs = [f"{tmp}.{os.path.basename(s)}.o" for s in srcs]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [_nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines],
               "-c", "-o", obj, src]
        return subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(srcs)) as ex:
        results = list(ex.map(compile_one, zip(srcs, objs)))
    try:
        for r in results:
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stderr}")
            if verbose:
                sys.stderr.write(r.stderr)
        r = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc link failed ({r.returncode}):\n{r.stderr}")
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
