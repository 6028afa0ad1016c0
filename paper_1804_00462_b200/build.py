"""Build the sm_100a extension in-tree: paper_1804_00462_b200/_lib/libsorsvd_b200.so.

Plain nvcc (no torch cpp_extension): the library has a C ABI
(include/sorsvd_b200.h) and no torch types, so it is loadable from C, C++,
ctypes or any FFI. Links the system NCCL (libnccl.so.2); inside a torch
process the already-loaded torch NCCL satisfies the same soname.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libsorsvd_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["sorsvd.cu", "host_rng.cpp"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h")))


def _deps():
    return [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "sorsvd_b200.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps() if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    # the library is stamped with the newest source time seen when the build started, so
    # an edit made while nvcc runs still marks it stale
    t_src = max(os.path.getmtime(p) for p in _deps() if os.path.exists(p))
    objs = []
    for src in SOURCES:
        obj = os.path.join(OUT_DIR, src + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        # SORSVD_OZ_LEVEL0=6: the 28-product cut of the Ozaki passes (default 5 = 34 products)
        if os.environ.get("SORSVD_OZ_LEVEL0"):
            cmd.insert(1, "-DOZ_LEVEL0=" + str(int(os.environ["SORSVD_OZ_LEVEL0"])))
        if src.endswith(".cpp"):
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-I", os.path.join(ROOT, "include"), "-c",
                   os.path.join(CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"], check=True)
    os.replace(tmp, LIB)
    os.utime(LIB, (t_src, t_src))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
