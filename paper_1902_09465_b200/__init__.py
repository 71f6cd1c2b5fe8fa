"""Python binding of libaknn.so -- the B200 hot path of adaptive k-NN (arXiv 1902.09465).

Argument marshalling only: every step of the path runs in the CUDA kernels of
``csrc/`` behind the C-ABI declared in ``include/aknn.h``; the names follow
that header.  There is no CPU fallback: importing this package without the
built library raises, and every call checks the library's status code.

Host API (numpy in, numpy out) and device API (torch CUDA tensors, current
torch stream) are both provided; torch is only used for device memory and
streams.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AKNN_LIB") or os.path.join(_HERE, "libaknn.so")  # AKNN_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)

AKNN_OK, AKNN_EINVAL, AKNN_ENOMEM, AKNN_ECUDA, AKNN_ENCCL, AKNN_EMAXROUNDS = 0, -1, -2, -3, -4, -5


class AknnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_lib.aknn_strerror(status).decode()}: {msg}")
        self.status = status


class Result(C.Structure):
    _fields_ = [("sets", C.c_void_p), ("dhat", C.c_void_p), ("counts", C.c_void_p),
                ("sums", C.c_void_p), ("evals", C.c_void_p), ("draws", C.c_void_p),
                ("rounds", C.c_void_p)]


class Opts(C.Structure):
    _fields_ = [("qi_offset", C.c_int32), ("max_rounds", C.c_int32), ("timing", C.c_int32),
                ("flags", C.c_int32), ("lead", C.c_int32), ("batch_queries", C.c_int32),
                ("growth", C.c_int32)]


FLAG_RADIX_SELECT = 1
FLAG_EXACT_ROWS = 2  # exact fallbacks as per-pair row streams instead of tensor-core tiles
FLAG_NO_TILES = 4  # every level gather through the work lists (no shared-memory tiles)
FLAG_EXACT_MMA_ALL = 8  # every tile with an exact fallback on the tensor cores
FLAG_SHARED_DRAWS = 16  # query-independent coordinate draws
FLAG_NO_LEVEL_MMA = 32  # shared draws without the tensor-core level GEMMs
FLAG_WITHOUT_REPLACEMENT = 64  # sampling without replacement (footnote 1 to P:120; reading R23)


class Stats(C.Structure):
    _fields_ = [("rounds", C.c_int32), ("query_batches", C.c_int32),
                ("kernel_launches", C.c_int64), ("pairs", C.c_int64), ("draws", C.c_int64),
                ("exact_fallbacks", C.c_int64), ("active_pair_rounds", C.c_int64),
                ("query_rounds", C.c_int64), ("blocked_query_rounds", C.c_int64),
                ("ms_total", C.c_double), ("ms_init", C.c_double), ("ms_select", C.c_double),
                ("ms_filter", C.c_double), ("ms_compact", C.c_double),
                ("ms_advance", C.c_double), ("ms_output", C.c_double),
                ("launches_init", C.c_int64), ("launches_select", C.c_int64),
                ("launches_filter", C.c_int64), ("launches_compact", C.c_int64),
                ("launches_advance", C.c_int64), ("launches_output", C.c_int64),
                ("philox_blocks", C.c_int64), ("graph_builds", C.c_int32), ("pad0", C.c_int32),
                ("ms_tiles", C.c_double), ("launches_tiles", C.c_int64), ("tile_blocks", C.c_int64),
                ("tile_draws", C.c_int64), ("level_mma_tiles", C.c_int64)]


class MergeResult(C.Structure):
    _fields_ = [("sets", C.c_void_p), ("dhat", C.c_void_p), ("thr_k", C.c_uint64),
                ("thr_kh", C.c_uint64), ("A", C.c_double), ("B", C.c_double),
                ("d1", C.c_int64), ("d2", C.c_int64), ("alpha_d2", C.c_double),
                ("stop", C.c_int32)]


SHARD_REC_BYTES = 16

_P = C.c_void_p
_I = C.c_int32
_L = C.c_int64
_sig = {
    "aknn_build": ([_P, _L, _I, C.POINTER(_P)], _I),
    "aknn_build_async": ([_P, _L, _I, _P, C.POINTER(_P)], _I),
    "aknn_build_shard": ([_P, _L, _L, _L, _I, _P, _I, _I, C.POINTER(_P)], _I),
    "aknn_nccl_unique_id": ([_P], _I),
    "aknn_set_timeout": ([_P, C.c_double], _I),
    "aknn_query": ([_P, _P, _I, _I, _I, C.c_double, C.c_uint64, _P, C.POINTER(Result)], _I),
    "aknn_query_ex": ([_P, _P, _I, _I, _I, C.c_double, C.c_uint64, _P, C.POINTER(Opts),
                       C.POINTER(Result)], _I),
    "aknn_query_async": ([_P, _P, _I, _I, _I, C.c_double, C.c_uint64, _P, C.POINTER(Opts),
                          C.POINTER(Result), _P], _I),
    "aknn_query_a1": ([_P, _P, _I, _I, _I, C.c_double, C.c_uint64, _P, C.POINTER(Opts),
                       C.POINTER(Result)], _I),
    "aknn_query_a1_device": ([_P, _P, _I, _I, _I, C.c_double, C.c_uint64, _P, C.POINTER(Opts),
                              C.POINTER(Result), _P], _I),
    "aknn_query_multi": ([C.POINTER(_P), _I, _P, _I, _I, _I, C.c_double, C.c_uint64, _P,
                          C.POINTER(Opts), C.POINTER(Result)], _I),
    "aknn_get_stats": ([_P, C.POINTER(Stats)], _I),
    "aknn_shard_summary_host": ([_P, _P, _L, _L, _L, _I, _I, _I, _P, _P], _I),
    "aknn_shard_merge_host": ([_P, _I, _L, _I, _I, _I, _P, C.POINTER(MergeResult)], _I),
    "aknn_exact": ([_P, _P, _I, _I, _P, _P], _I),
    "aknn_exact_async": ([_P, _P, _I, _I, _P, _P, _P], _I),
    "aknn_alpha_table": ([_I, _L, C.c_double, C.c_double, _I, _P], _I),
    "aknn_index_n_local": ([_P], _L),
    "aknn_index_n_global": ([_P], _L),
    "aknn_index_dim": ([_P], _I),
    "aknn_free": ([_P], None),
    "aknn_strerror": ([_I], C.c_char_p),
    "aknn_last_error": ([], C.c_char_p),
}
for _name, (_args, _ret) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _ret

EXPORTS = tuple(_sig)


def _check(status: int):
    if status not in (AKNN_OK,):
        raise AknnError(status, (_lib.aknn_last_error() or b"").decode())


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def alpha_table(n: int, delta: float, d: int, kind: str = "theory", c_alpha: float = 1.0) -> np.ndarray:
    """aknn_alpha_table: kind 'theory' = footnote 2, 'experimental' = §5."""
    out = np.zeros(d + 1, np.float64)
    _check(_lib.aknn_alpha_table(0 if kind == "theory" else 1, n, delta, c_alpha, d, _ptr(out)))
    return out


def query_multi(shards, queries, k: int, h: int, delta: float, seed: int = 0, alpha=None, *,
                counts: bool = True, sums: bool = False, dhat: bool = True, max_rounds: int = 0,
                qi_offset: int = 0, timing: bool = False, flags: int = 0, lead: int = 1,
                batch_queries: int = 0, growth: int = 1) -> dict:
    """aknn_query_multi: one query batch over shard indices on the current device.

    ``shards`` are Index objects built with ``Index(rows, n_global=..., offset=...)``
    tiling [0, n_global) in order; counts/sums come back with n_global columns."""
    Q = np.ascontiguousarray(np.atleast_2d(queries), np.uint8)
    q, d = Q.shape
    if not shards:
        raise AknnError(AKNN_EINVAL, "need at least one shard")
    if d != shards[0].d:
        raise AknnError(AKNN_EINVAL, f"query dimension {d} != index dimension {shards[0].d}")
    n = shards[0].n_global
    kh = k + h
    out = dict(sets=np.zeros((q, kh), np.int32),
               dhat=np.zeros((q, kh), np.float64) if dhat else None,
               counts=np.zeros((q, n), np.int32) if counts else None,
               sums=np.zeros((q, n), np.int64) if sums else None,
               evals=np.zeros(q, np.int64), draws=np.zeros(q, np.int64),
               rounds=np.zeros(q, np.int32))
    res = Result(*[_ptr(out[f]) for f, _ in Result._fields_])
    al = None if alpha is None else np.ascontiguousarray(alpha, np.float64)
    if al is not None and al.shape != (d + 1,):
        raise AknnError(AKNN_EINVAL, f"alpha must have d+1={d + 1} entries")
    arr = (_P * len(shards))(*[s._h for s in shards])
    opts = Opts(qi_offset, max_rounds, 1 if timing else 0, flags, lead, batch_queries, growth)
    st = _lib.aknn_query_multi(arr, len(shards), _ptr(Q), q, k, h, delta, seed & (2**64 - 1),
                               _ptr(al), C.byref(opts), C.byref(res))
    out["status"] = st
    if st != AKNN_EMAXROUNDS:
        _check(st)
    return out


def shard_summary_host(S, lvl, offset: int, n_global: int, d: int, k: int, h: int,
                       alpha) -> np.ndarray:
    """aknn_shard_summary_host: one query's shard summary as (k+h+1)*16 raw bytes."""
    S = np.ascontiguousarray(S, np.int32)
    lvl = np.ascontiguousarray(lvl, np.uint8)
    al = np.ascontiguousarray(alpha, np.float64)
    out = np.zeros((k + h + 1) * SHARD_REC_BYTES, np.uint8)
    _check(_lib.aknn_shard_summary_host(_ptr(S), _ptr(lvl), S.shape[0], offset, n_global, d, k, h,
                                        _ptr(al), _ptr(out)))
    return out


def shard_merge_host(recs, world: int, n_global: int, d: int, k: int, h: int, alpha) -> dict:
    """aknn_shard_merge_host on the concatenated summaries of `world` shards."""
    recs = np.ascontiguousarray(recs, np.uint8)
    al = np.ascontiguousarray(alpha, np.float64)
    sets = np.zeros(k + h, np.int32)
    dh = np.zeros(k + h, np.float64)
    r = MergeResult(sets.ctypes.data, dh.ctypes.data, 0, 0, 0.0, 0.0, 0, 0, 0.0, 0)
    _check(_lib.aknn_shard_merge_host(_ptr(recs), world, n_global, d, k, h, _ptr(al), C.byref(r)))
    return dict(sets=sets, dhat=dh, thr_k=r.thr_k, thr_kh=r.thr_kh, A=r.A, B=r.B, d1=r.d1,
                d2=r.d2, alpha_d2=r.alpha_d2, stop=bool(r.stop))


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(_lib.aknn_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def _torch():
    import torch
    return torch


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


class Index:
    """aknn_index: a device copy of the point set X (uint8 [n][d])."""

    def __init__(self, points, *, n_global: Optional[int] = None, offset: int = 0,
                 nccl_id: Optional[bytes] = None, rank: int = 0, world: int = 1, stream=None):
        h = _P()
        if isinstance(points, np.ndarray):
            pts = np.ascontiguousarray(points, np.uint8)
            n, d = pts.shape
            if n_global is None and world == 1 and offset == 0:
                _check(_lib.aknn_build(_ptr(pts), n, d, C.byref(h)))
            else:
                idbuf = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
                _check(_lib.aknn_build_shard(_ptr(pts), n, n_global or n, offset, d,
                                             None if idbuf is None else C.cast(idbuf, C.c_void_p),
                                             rank, world, C.byref(h)))
        else:
            torch = _torch()
            assert points.is_cuda and points.dtype == torch.uint8 and points.dim() == 2
            pts = points.contiguous()
            n, d = pts.shape
            _check(_lib.aknn_build_async(_ptr(pts), n, d, _stream_ptr(stream), C.byref(h)))
            (torch.cuda.current_stream() if stream is None else stream).synchronize()
        self._h = h
        self.n_local = int(_lib.aknn_index_n_local(h))
        self.n_global = int(_lib.aknn_index_n_global(h))
        self.d = int(_lib.aknn_index_dim(h))

    def set_timeout(self, timeout_ms: float):
        """aknn_set_timeout: deadline of a sharded round (peer failure detection)."""
        _check(_lib.aknn_set_timeout(self._h, float(timeout_ms)))

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.aknn_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # ------------------------------------------------------------------ query
    def query(self, queries, k: int, h: int, delta: float, seed: int = 0, alpha=None, *,
              counts: bool = True, sums: bool = False, dhat: bool = True, max_rounds: int = 0,
              qi_offset: int = 0, timing: bool = False, out: Optional[dict] = None,
              flags: int = 0, schedule: str = "br", lead: int = 1, batch_queries: int = 0,
              growth: int = 1) -> dict:
        """aknn_query_ex on host arrays; returns numpy arrays.

        ``schedule="a1"`` runs the literal Algorithm 1 instead (aknn_query_a1;
        ``rounds`` then counts iterations and ``max_rounds`` caps them).
        ``out`` may pass preallocated (e.g. pinned) host arrays with the keys of the
        returned dict; a key mapped to None skips that output."""
        if schedule not in ("br", "a1"):
            raise AknnError(AKNN_EINVAL, f"schedule must be 'br' or 'a1', not {schedule!r}")
        Q = np.ascontiguousarray(np.atleast_2d(queries), np.uint8)
        q, d = Q.shape
        if d != self.d:
            raise AknnError(AKNN_EINVAL, f"query dimension {d} != index dimension {self.d}")
        kh = k + h
        if out is None:
            out = dict(sets=np.zeros((q, kh), np.int32),
                       dhat=np.zeros((q, kh), np.float64) if dhat else None,
                       counts=np.zeros((q, self.n_local), np.int32) if counts else None,
                       sums=np.zeros((q, self.n_local), np.int64) if sums else None,
                       evals=np.zeros(q, np.int64), draws=np.zeros(q, np.int64),
                       rounds=np.zeros(q, np.int32))
        else:
            want = dict(sets=((q, kh), np.int32), dhat=((q, kh), np.float64),
                        counts=((q, self.n_local), np.int32), sums=((q, self.n_local), np.int64),
                        evals=((q,), np.int64), draws=((q,), np.int64), rounds=((q,), np.int32))
            for key, (shape, dt) in want.items():
                a = out.get(key)
                if a is None:
                    if key == "sets":
                        raise AknnError(AKNN_EINVAL, "out['sets'] is required")
                    out[key] = None
                elif a.shape != shape or a.dtype != dt or not a.flags.c_contiguous:
                    raise AknnError(AKNN_EINVAL, f"out[{key!r}] must be C-contiguous {dt.__name__}{shape}")
        res = Result(*[_ptr(out[f]) for f, _ in Result._fields_])
        al = None if alpha is None else np.ascontiguousarray(alpha, np.float64)
        if al is not None and al.shape != (self.d + 1,):
            raise AknnError(AKNN_EINVAL, f"alpha must have d+1={self.d + 1} entries")
        opts = Opts(qi_offset, max_rounds, 1 if timing else 0, flags, lead, batch_queries, growth)
        fn = _lib.aknn_query_a1 if schedule == "a1" else _lib.aknn_query_ex
        st = fn(self._h, _ptr(Q), q, k, h, delta, seed & (2**64 - 1), _ptr(al), C.byref(opts),
                C.byref(res))
        out["status"] = st
        if st != AKNN_EMAXROUNDS:
            _check(st)
        return out

    def query_device(self, queries, k: int, h: int, delta: float, seed: int = 0, alpha=None, *,
                     counts: bool = False, sums: bool = False, dhat: bool = True,
                     max_rounds: int = 0, qi_offset: int = 0, timing: bool = False,
                     stream=None, out: Optional[dict] = None, flags: int = 0,
                     schedule: str = "br", lead: int = 1, batch_queries: int = 0,
                     growth: int = 1) -> dict:
        """aknn_query_async on torch CUDA tensors (current stream); returns device tensors.

        ``schedule="a1"``: the literal Algorithm 1 (aknn_query_a1_device; waits for the
        stream before returning)."""
        if schedule not in ("br", "a1"):
            raise AknnError(AKNN_EINVAL, f"schedule must be 'br' or 'a1', not {schedule!r}")
        torch = _torch()
        if not (queries.is_cuda and queries.dtype == torch.uint8 and queries.dim() == 2):
            raise AknnError(AKNN_EINVAL, "queries must be a 2-D uint8 CUDA tensor")
        Q = queries.contiguous()
        q, d = Q.shape
        if d != self.d:
            raise AknnError(AKNN_EINVAL, f"query dimension {d} != index dimension {self.d}")
        kh = k + h
        dev = Q.device
        if out is None:
            out = dict(sets=torch.empty((q, kh), dtype=torch.int32, device=dev),
                       dhat=torch.empty((q, kh), dtype=torch.float64, device=dev) if dhat else None,
                       counts=torch.empty((q, self.n_local), dtype=torch.int32, device=dev) if counts else None,
                       sums=torch.empty((q, self.n_local), dtype=torch.int64, device=dev) if sums else None,
                       evals=torch.empty(q, dtype=torch.int64, device=dev),
                       draws=torch.empty(q, dtype=torch.int64, device=dev),
                       rounds=torch.empty(q, dtype=torch.int32, device=dev))
        res = Result(*[_ptr(out.get(f)) for f, _ in Result._fields_])
        al = None
        if alpha is not None:
            al = alpha if (hasattr(alpha, "is_cuda") and alpha.is_cuda) else \
                torch.as_tensor(np.ascontiguousarray(alpha, np.float64)).to(dev)
            if al.dtype != torch.float64 or al.numel() != self.d + 1 or not al.is_contiguous():
                raise AknnError(AKNN_EINVAL, f"alpha must be a contiguous float64 tensor of d+1={self.d + 1} entries")
        opts = Opts(qi_offset, max_rounds, 1 if timing else 0, flags, lead, batch_queries, growth)
        fn = _lib.aknn_query_a1_device if schedule == "a1" else _lib.aknn_query_async
        st = fn(self._h, _ptr(Q), q, k, h, delta, seed & (2**64 - 1), _ptr(al), C.byref(opts),
                C.byref(res), _stream_ptr(stream))
        out["status"] = st
        if st != AKNN_EMAXROUNDS:
            _check(st)
        return out

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.aknn_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    # ------------------------------------------------------------------ exact
    def exact(self, queries, k: int):
        """aknn_exact: exact k nearest by (sum (a-b)^2, id); host arrays."""
        Q = np.ascontiguousarray(np.atleast_2d(queries), np.uint8)
        q = Q.shape[0]
        if Q.shape[1] != self.d:
            raise AknnError(AKNN_EINVAL, f"query dimension {Q.shape[1]} != index dimension {self.d}")
        idx = np.zeros((q, k), np.int32)
        dist = np.zeros((q, k), np.int32)
        _check(_lib.aknn_exact(self._h, _ptr(Q), q, k, _ptr(idx), _ptr(dist)))
        return idx, dist

    def exact_device(self, queries, k: int, stream=None, out=None):
        """aknn_exact_async on torch CUDA tensors."""
        torch = _torch()
        if not (queries.is_cuda and queries.dtype == torch.uint8 and queries.dim() == 2
                and queries.shape[1] == self.d):
            raise AknnError(AKNN_EINVAL, f"queries must be a uint8 CUDA tensor [q][{self.d}]")
        Q = queries.contiguous()
        q = Q.shape[0]
        if out is None:
            out = (torch.empty((q, k), dtype=torch.int32, device=Q.device),
                   torch.empty((q, k), dtype=torch.int32, device=Q.device))
        _check(_lib.aknn_exact_async(self._h, _ptr(Q), q, k, _ptr(out[0]), _ptr(out[1]),
                                     _stream_ptr(stream)))
        return out
