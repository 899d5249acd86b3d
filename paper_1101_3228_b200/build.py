"""Build libqtree_cuda.so in-tree for sm_100a (explicit nvcc, no JIT cache).

    python -m paper_1101_3228_b200.build [--force]

The shared library lands in paper_1101_3228_b200/lib/ so it travels with the
repo snapshot to the GPU box; nothing is installed into site-packages.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libqtree_cuda.so")
# development hook: load a variant build (e.g. other -D tuning flags) instead
LIB = os.environ.get("QT_LIB_VARIANT") or LIB

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "-shared"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libqtree_cuda.so")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps() -> list[str]:
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) +
                              glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "qtree_cuda.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if os.environ.get("QT_LIB_VARIANT"):
        return LIB
    if not force and up_to_date():
        return LIB
    import fcntl
    os.makedirs(LIB_DIR, exist_ok=True)
    # one builder at a time (torchrun starts one process per GPU, each may call build())
    with open(os.path.join(LIB_DIR, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and up_to_date():
            return LIB
        tmp = f"{LIB}.tmp{os.getpid()}"
        # one nvcc per translation unit in parallel (no relocatable device code:
        # every kernel lives in one TU), then one host link
        from concurrent.futures import ThreadPoolExecutor
        # objects persist in lib/obj (git-ignored): a TU is recompiled only when
        # it or any header is newer than its object
        objdir = os.path.join(LIB_DIR, "obj")
        os.makedirs(objdir, exist_ok=True)
        compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
        hdr_t = max(os.path.getmtime(d) for d in deps() if not d.endswith(".cu"))

        def compile_one(src: str) -> str:
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            if (not force and os.path.exists(obj) and
                    os.path.getmtime(obj) >= max(hdr_t, os.path.getmtime(src))):
                return obj
            tmpo = f"{obj}.tmp{os.getpid()}"
            cmd = [nvcc(), *ARCH, *compile_flags, "-c", "-o", tmpo, src]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            os.replace(tmpo, obj)
            return obj

        try:
            with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
                objs = list(ex.map(compile_one, sources()))
            cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-ldl"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            os.replace(tmp, LIB)
        finally:
            if os.path.exists(tmp):
                os.remove(tmp)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
