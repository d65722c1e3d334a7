"""Build libftn.so (sm_100a) in-tree with nvcc.

    python -m paper_2409_18824_b200.build

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false (no FMA
contraction anywhere: DESIGN.md R#19), static cudart, linked against the NCCL
2.28 that torch ships (the system 2.27 has the same SONAME).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "ftn")
LIB = os.path.join(PKG, "libftn.so")
SOURCES = ["desc", "elemental", "reduce", "reduce_dim", "transpose", "matmul", "stencil", "stencil_tb", "stencil_wq", "stencil3d_tb", "stencil3d_wr", "advection", "tra_adv", "dist"]


def nccl_root() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch's NCCL) not found")
    return list(spec.submodule_search_locations)[0]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def flags():
    nccl = nccl_root()
    return ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
            "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nccl, "include")]


def _compile(name: str) -> str:
    src = os.path.join(CSRC, name + ".cu")
    obj = os.path.join(BUILD, name + ".o")
    deps = [src, os.path.join(CSRC, "ftn_internal.cuh"), os.path.join(ROOT, "include", "ftn.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [nvcc()] + flags() + ["-Xptxas", "-v", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(BUILD, name + ".ptxas.log"), "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}.cu:\n{r.stderr[-4000:]}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    nccl_lib = os.path.join(nccl_root(), "lib")
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp"] + objs + [
        "-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nccl_lib, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
