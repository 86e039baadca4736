"""Build libchunkstar_b200.so (sm_100a) in-tree, and the C oracle for tests.

``python -m paper_2108_05818_b200._build`` or ``__graft_entry__.build()``.
The CUDA sources are compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3``; the host
Adam with ``g++ -O3 -fopenmp -ffp-contract=off``.  Rebuilds only when a
source or header is newer than the library.
"""

import os
import subprocess
import sys
from typing import List

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libchunkstar_b200.so")

CUDA_SOURCES = ["adam.cu", "adam_tma.cu", "sumsq.cu", "pack.cu", "xent.cu", "layernorm.cu",
                "embed.cu"]
HOST_SOURCES = ["host_adam.cpp", "host_embed.cpp", "capi.cpp", "gemm_gelu.cpp", "comm.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SOURCES = ["cs_oracle.c"]
ORACLE_LIB = os.path.join(ORACLE_DIR, "_build", "libcs_oracle.so")


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale(target: str, deps: List[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: List[str], verbose: bool) -> None:
    if verbose:
        print("+", " ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("build step failed (%d): %s\n%s%s"
                           % (res.returncode, " ".join(cmd), res.stdout, res.stderr))
    if verbose and (res.stdout.strip() or res.stderr.strip()):
        print(res.stdout + res.stderr, flush=True)


def build_library(verbose: bool = False, force: bool = False) -> str:
    headers = [os.path.join(INCLUDE, "chunkstar_b200.h"),
               os.path.join(CSRC, "cs_internal.h")]
    sources = [os.path.join(CSRC, s) for s in CUDA_SOURCES + HOST_SOURCES]
    if not force and not _stale(LIB, sources + headers + [__file__]):
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    common = ["-I", INCLUDE, "-I", CSRC]
    for src in CUDA_SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        _run([_nvcc(), *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xptxas", "-v",
              "-Xcompiler", "-fPIC", *common, "-c", os.path.join(CSRC, src), "-o", obj],
             verbose)
        objs.append(obj)
    cuda_home = os.path.dirname(os.path.dirname(os.path.realpath(_nvcc()))) \
        if os.path.sep in _nvcc() else "/usr/local/cuda"
    for src in HOST_SOURCES:
        obj = os.path.join(BUILD, src + ".o")
        _run(["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off",
              *common, "-I", os.path.join(cuda_home, "include"), "-c",
              os.path.join(CSRC, src), "-o", obj], verbose)
        objs.append(obj)
    tmp = LIB + ".tmp"
    _run([_nvcc(), *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs,
          "-Xcompiler", "-fopenmp", "-lgomp", "-lcublasLt", "-ldl"], verbose)
    os.replace(tmp, LIB)
    return LIB


def build_oracle(verbose: bool = False, force: bool = False) -> str:
    """The C restatement used ONLY by tests / smoke / bench cpu_baseline."""
    sources = [os.path.join(ORACLE_DIR, s) for s in ORACLE_SOURCES]
    if not all(os.path.exists(s) for s in sources):
        return ""
    if not force and not _stale(ORACLE_LIB, sources + [__file__]):
        return ORACLE_LIB
    os.makedirs(os.path.dirname(ORACLE_LIB), exist_ok=True)
    tmp = ORACLE_LIB + ".tmp"
    _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
          "-fno-fast-math", "-o", tmp, *sources, "-lm"], verbose)
    os.replace(tmp, ORACLE_LIB)
    return ORACLE_LIB


if __name__ == "__main__":
    v = "-v" in sys.argv
    f = "-f" in sys.argv
    print(build_library(verbose=v, force=f))
    print(build_oracle(verbose=v, force=f))
