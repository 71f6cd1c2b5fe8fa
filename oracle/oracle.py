"""ctypes wrapper of the CPU oracle (oracle/aknn_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py may import this
module.  The product package ``paper_1902_09465_b200`` never does.

Argument marshalling only; every computation happens in the C file, whose
functions cite PAPER.md / SPEC.md line by line.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aknn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ENOMEM, EMAXROUNDS, EINTERNAL = 0, -1, -2, -5, -9


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, -O2 -ffp-contract=off, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_lemire.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_lemire.restype = C.c_uint32
        L.orc_lemire_histogram.argtypes = [C.c_uint32, P]
        L.orc_draw_index.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int64, C.c_uint32]
        L.orc_draw_index.restype = C.c_uint32
        L.orc_alpha_theory.argtypes = [C.c_int64, C.c_double, C.c_int32, P]
        L.orc_alpha_experimental.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_int32, P]
        L.orc_bruteforce.argtypes = [P, C.c_int64, C.c_int32, P, C.c_int32, C.c_int32, P, P]
        L.orc_round_step.argtypes = [C.c_int64, C.c_int32, P, P, C.c_int32, C.c_int32, P, P,
                                     P, P, P, P, P]
        L.orc_query_br.argtypes = [P, C.c_int64, C.c_int32, P, C.c_int32, P, C.c_int64,
                                   C.c_int32, C.c_int32, C.c_uint64, P, C.c_int32,
                                   C.c_int32, C.c_int32, C.c_int32, P, P, P, P, P, P, P]
        L.orc_next_count.argtypes = [C.c_int64, C.c_int32]
        L.orc_next_count.restype = C.c_int64
        L.orc_query_a1.argtypes = [P, C.c_int64, C.c_int32, P, C.c_int32, C.c_int32,
                                   C.c_int32, C.c_uint64, P, C.c_int64, C.c_int32, P, P, P, P, P, P]
        L.orc_wor_radix.argtypes = [C.c_uint32, P, P]
        L.orc_wor_keys.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, P]
        L.orc_feistel.restype = C.c_uint32
        L.orc_feistel.argtypes = [P, C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_wor_index.restype = C.c_uint32
        L.orc_wor_index.argtypes = [P, C.c_uint32, C.c_uint32]
        L.orc_wor_perm.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def lemire(w: int, d: int) -> int:
    return int(lib().orc_lemire(w, d))


def lemire_histogram(d: int) -> np.ndarray:
    h = np.zeros(d, np.uint64)
    lib().orc_lemire_histogram(d, _p(h))
    return h


def draw_index(seed: int, qi: int, i: int, t: int, d: int) -> int:
    return int(lib().orc_draw_index(seed, qi, i, t, d))


def alpha_theory(n: int, delta: float, d: int) -> np.ndarray:
    a = np.zeros(d + 1, np.float64)
    rc = lib().orc_alpha_theory(n, delta, d, _p(a))
    if rc != OK:
        raise ValueError(f"alpha_theory undefined for n={n}, delta={delta} (rc={rc})")
    return a


def alpha_experimental(n: int, delta: float, d: int, c_alpha: float) -> np.ndarray:
    a = np.zeros(d + 1, np.float64)
    rc = lib().orc_alpha_experimental(n, delta, c_alpha, d, _p(a))
    if rc != OK:
        raise ValueError(f"alpha_experimental: bad arguments (rc={rc})")
    return a


def bruteforce(X: np.ndarray, Q: np.ndarray, k: int):
    X = np.ascontiguousarray(X, np.uint8)
    Q = np.ascontiguousarray(np.atleast_2d(Q), np.uint8)
    n, d = X.shape
    q = Q.shape[0]
    idx = np.zeros((q, k), np.int32)
    dist = np.zeros((q, k), np.int64)
    rc = lib().orc_bruteforce(_p(X), n, d, _p(Q), q, k, _p(idx), _p(dist))
    if rc != OK:
        raise ValueError(f"bruteforce rc={rc}")
    return idx, dist


def round_step(S, T, d: int, k: int, h: int, alpha, want_active: bool = True):
    S = np.ascontiguousarray(S, np.int64)
    T = np.ascontiguousarray(T, np.int32)
    alpha = np.ascontiguousarray(alpha, np.float64)
    n = S.shape[0]
    order = np.zeros(n, np.int32)
    d1 = C.c_int32()
    d2 = C.c_int32()
    A = C.c_double()
    B = C.c_double()
    act = np.zeros(n, np.uint8) if want_active else None
    rc = lib().orc_round_step(n, d, _p(S), _p(T), k, h, _p(alpha), _p(order), C.byref(d1),
                              C.byref(d2), C.byref(A), C.byref(B), _p(act))
    if rc < 0:
        raise ValueError(f"round_step rc={rc}")
    return dict(stop=bool(rc), order=order, d1=d1.value, d2=d2.value, A=A.value, B=B.value,
                active=None if act is None else act.astype(bool))


SHARED_QI = 0xFFFFFFFF  # the counter word of query-independent draws


def query_br(X, Q, k: int, h: int, seed: int, alpha, qids=None, id_offset: int = 0,
             max_rounds: int = 0, want_counts: bool = True, want_sums: bool = False,
             shared_draws: bool = False, without_replacement: bool = False, lead: int = 1,
             growth: int = 1):
    """Batched round rule BR, one query at a time.  shared_draws:
    every query's counter word is SHARED_QI, i.e. arm i's t-th coordinate is the same
    for all queries; each query alone is unchanged in law."""
    X = np.ascontiguousarray(X, np.uint8)
    Q = np.ascontiguousarray(np.atleast_2d(Q), np.uint8)
    alpha = np.ascontiguousarray(alpha, np.float64)
    n, d = X.shape
    q = Q.shape[0]
    assert Q.shape[1] == d and alpha.shape[0] == d + 1
    qids = np.arange(q, dtype=np.int32) if qids is None else np.ascontiguousarray(qids, np.int32)
    if shared_draws:
        qids = np.full(q, SHARED_QI, np.uint32).view(np.int32)
    kh = k + h
    out = dict(
        sets=np.zeros((q, kh), np.int32), dhat=np.zeros((q, kh), np.float64),
        counts=np.zeros((q, n), np.int32) if want_counts else None,
        sums=np.zeros((q, n), np.int64) if want_sums else None,
        evals=np.zeros(q, np.int64), draws=np.zeros(q, np.int64), rounds=np.zeros(q, np.int32))
    rc = lib().orc_query_br(_p(X), n, d, _p(Q), q, _p(qids), id_offset, k, h,
                            C.c_uint64(seed & (2**64 - 1)), _p(alpha), max_rounds,
                            1 if without_replacement else 0, lead, growth, _p(out["sets"]), _p(out["dhat"]), _p(out["counts"]),
                            _p(out["sums"]), _p(out["evals"]), _p(out["draws"]),
                            _p(out["rounds"]))
    out["status"] = rc
    if rc not in (OK, EMAXROUNDS):
        raise ValueError(f"query_br rc={rc}")
    return out


def next_count(T: int, m: int) -> int:
    """The next per-arm sample count after T under the growth-m schedule (reading R25)."""
    return int(lib().orc_next_count(T, m))


def query_a1(X, x, k: int, h: int, seed: int, alpha, qi: int = 0, max_iters: int = 0,
             without_replacement: bool = False):
    """Literal Algorithm 1 for one query; tiny inputs only."""
    X = np.ascontiguousarray(X, np.uint8)
    x = np.ascontiguousarray(x, np.uint8).reshape(-1)
    alpha = np.ascontiguousarray(alpha, np.float64)
    n, d = X.shape
    kh = k + h
    out = dict(set=np.zeros(kh, np.int32), counts=np.zeros(n, np.int32),
               sums=np.zeros(n, np.int64))
    ev, dr, it = C.c_int64(), C.c_int64(), C.c_int64()
    rc = lib().orc_query_a1(_p(X), n, d, _p(x), qi, k, h, C.c_uint64(seed & (2**64 - 1)),
                            _p(alpha), max_iters, 1 if without_replacement else 0, _p(out["set"]), _p(out["counts"]),
                            _p(out["sums"]), C.byref(ev), C.byref(dr), C.byref(it))
    if rc not in (OK, EMAXROUNDS):
        raise ValueError(f"query_a1 rc={rc}")
    out.update(status=rc, evals=ev.value, draws=dr.value, iters=it.value)
    return out


# ---- sampling without replacement (footnote 1 to P:120; reading R23) ----
def wor_radix(d: int):
    """(a, b) of the mixed-radix Feistel domain Z_a x Z_b: a = ceil(sqrt d), b = ceil(d / a)."""
    a, b = C.c_uint32(), C.c_uint32()
    lib().orc_wor_radix(d, C.byref(a), C.byref(b))
    return a.value, b.value


def wor_keys(seed: int, qi: int, i: int) -> np.ndarray:
    k = np.zeros(4, np.uint32)
    lib().orc_wor_keys(C.c_uint64(seed & (2**64 - 1)), qi, i, _p(k))
    return k


def feistel(keys, a: int, b: int, x: int) -> int:
    k = np.ascontiguousarray(keys, np.uint32)
    return int(lib().orc_feistel(_p(k), a, b, x))


def wor_index(keys, d: int, t: int) -> int:
    k = np.ascontiguousarray(keys, np.uint32)
    return int(lib().orc_wor_index(_p(k), d, t))


def wor_perm(seed: int, qi: int, i: int, d: int) -> np.ndarray:
    """pi(0..d-1) of arm (qi, i): the order in which it samples its coordinates."""
    out = np.zeros(d, np.uint32)
    lib().orc_wor_perm(C.c_uint64(seed & (2**64 - 1)), qi, i, d, _p(out))
    return out
