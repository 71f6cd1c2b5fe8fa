"""Compile libaknn.so in-tree for sm_100a (nvcc; no JIT cache, no torch extension).

The library links the same libnccl that torch loads (the pip nvidia-nccl wheel),
so one process never holds two NCCL copies.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libaknn.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # the copy torch loads
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except Exception:
        pass
    return None


def nvcc_cmd(out=LIB, extra=()):
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-ffp-contract=off", "-shared", "-I", os.path.join(ROOT, "include"),
           "-o", out, *srcs, *extra]
    nccl = _nccl_dirs()
    if nccl:
        inc, lib = nccl
        cmd += ["-DAKNN_WITH_NCCL", "-I", inc, "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    return cmd


def sources_newer_than(path):
    if not os.path.exists(path):
        return True
    t = os.path.getmtime(path)
    deps = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "aknn.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


PROBES_SRC = os.path.join(ROOT, "tools", "probes.cu")
PROBES_LIB = os.path.join(ROOT, "tools", "libprobes.so")


def build_probes(force: bool = False, verbose: bool = True) -> str:
    """tools/libprobes.so: roofline microbenchmarks used by bench.py (not the product)."""
    if force or not os.path.exists(PROBES_LIB) or os.path.getmtime(PROBES_LIB) < os.path.getmtime(PROBES_SRC):
        cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
               "-o", PROBES_LIB, PROBES_SRC]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    return PROBES_LIB


def build(force: bool = False, verbose: bool = True) -> str:
    if force or sources_newer_than(LIB):
        cmd = nvcc_cmd()
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    build_probes(force, verbose)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
