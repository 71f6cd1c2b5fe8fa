"""Measure the roofline denominators of the hot kernels on this GPU (tools/libprobes.so)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "libprobes.so")


def load():
    L = C.CDLL(LIB)
    L.probe_philox.argtypes = [C.c_int, C.c_longlong, C.c_uint32, C.c_int]
    L.probe_philox.restype = C.c_double
    L.probe_gather.argtypes = [C.c_int, C.c_int, C.c_ulonglong, C.c_int]
    L.probe_gather.restype = C.c_double
    L.probe_shared.argtypes = [C.c_int, C.c_int, C.c_int]
    L.probe_shared.restype = C.c_double
    return L


def philox_blocks_per_s(L, d=784, sms=148):
    threads = sms * 2048
    bpt = 512
    ms = L.probe_philox(threads, bpt, d, 5)
    return threads * bpt / (ms / 1e3) if ms > 0 else None


def shared_draws_per_s(L, sms=148):
    """Ceiling of the shared-draw tile gathers: (query, point) draws per second."""
    blocks, iters = sms * 3, 64
    ms = L.probe_shared(blocks, iters, 5)
    return blocks * 256 * iters * 256 / (ms / 1e3) if ms > 0 else None


def gather_sectors_per_s(L, footprint, sms=148):
    b = 1
    while b < footprint:
        b <<= 1
    threads = sms * 2048
    lpt = 256
    ms = L.probe_gather(threads, lpt, b, 5)
    return (threads * lpt / (ms / 1e3) if ms > 0 else None), b


if __name__ == "__main__":
    import torch  # noqa: F401  (CUDA context)
    torch.cuda.init()
    L = load()
    out = {"philox_blocks_per_s_d784": philox_blocks_per_s(L), "shared_draws_per_s": shared_draws_per_s(L)}
    for fp in (47_040_000, 1 << 30):
        r, b = gather_sectors_per_s(L, fp)
        out[f"gather_loads_per_s_{b >> 20}MiB"] = r
    print(json.dumps(out))
