"""Builds libhipattn.so (the C-ABI library) in-tree with nvcc for sm_100a only."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libhipattn.so")
# Debug variant (test infrastructure, SURVEY 8(c) C-2 replay parity): the product objects with
# mask_tc.cu rebuilt under -DHIPATTN_DEBUG_SCORES (the tcgen05 mask kernel dumps its branch scores).
DEBUG_LIB = os.path.join(PKG, "libhipattn_debug.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG, "csrc", "*.h")) + [
        os.path.join(ROOT, "include", "hip_attn.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in deps())


def build(force: bool = False, verbose: bool = False, extra=()) -> str:
    """One nvcc -c per source in parallel (objects under build/), then one nvcc link into the .so."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), *extra]
    if verbose:
        flags.insert(1, "-Xptxas=-v")

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = flags + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-o", LIB + ".tmp", *objs])
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_debug(force: bool = False) -> str:
    """libhipattn_debug.so: build() first, then mask_tc.cu again with -DHIPATTN_DEBUG_SCORES, linked
    with the other product objects."""
    build(force=False)
    if not force and os.path.exists(DEBUG_LIB) and os.path.getmtime(DEBUG_LIB) >= max(os.path.getmtime(f) for f in deps()):
        return DEBUG_LIB
    objdir = os.path.join(ROOT, "build", "obj")
    dbg_obj = os.path.join(ROOT, "build", "mask_tc_debug.o")
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
                           "-DHIPATTN_DEBUG_SCORES", "-c", os.path.join(PKG, "csrc", "mask_tc.cu"), "-o", dbg_obj])
    objs = [os.path.join(objdir, os.path.basename(src) + ".o") for src in sources()
            if os.path.basename(src) != "mask_tc.cu"] + [dbg_obj]
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-o", DEBUG_LIB + ".tmp", *objs])
    os.replace(DEBUG_LIB + ".tmp", DEBUG_LIB)
    return DEBUG_LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
