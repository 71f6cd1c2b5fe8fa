"""The SURVEY.md §8(d) parity set on the GPU box: every query of configs 2, 3 and 4 at
their BASELINE sizes (1,000 / 256 / 128 queries) through the bench's launch path
(aknn_query_async on device buffers, the whole batch in one call, graph-launched round
loop), compared with the CPU oracle query by query -- candidate sets, d_hat (0 ulp),
per-pair counts T_i and sums S_i over all n arms, draws, evals, rounds -- and config 5
at its full 8,000,000 points as 8 point shards of 1,000,000 on one GPU
(aknn_query_multi: the sharded kernels and merge of the N = 8 run) on sampled queries.

    python tools/parity_set.py [--configs 2,3,4,5] [--c5-queries 4] [--out profiles/r02_parity_set.json]

The oracle runs one single-threaded process per host core over disjoint queries (fork;
the oracle is test infrastructure, called here as the checker).  Result: a JSON record
per config with the number of queries compared and identical, and any mismatches."""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

KEYS = ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds")
_W = {}


def _orc_one(a):
    import oracle.oracle as orc
    X, Q, cfg, al = _W["X"], _W["Q"], _W["cfg"], _W["alpha"]
    r = orc.query_br(X, Q[a:a + 1], cfg.k, cfg.h, cfg.seed, al, qids=np.array([a], np.int32),
                     want_counts=True, want_sums=_W["sums"])
    return a, {k: (None if r[k] is None else r[k][0]) for k in KEYS}


def _compare(got, ref, a, keys):
    bad = []
    for k in keys:
        g, r = got[k][a], ref[k]
        if r is None:
            continue
        if not np.array_equal(np.asarray(g), np.asarray(r)):
            bad.append(k)
    return bad


def run_config(i, cores, nq=None):
    import torch
    import oracle.oracle as orc
    import paper_1902_09465_b200 as ak
    cfg = synth.config(i)
    X, Q = synth.points(cfg), synth.queries(cfg)
    if nq:
        Q = Q[:nq]
    q = Q.shape[0]
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    t0 = time.perf_counter()
    ix = ak.Index(torch.from_numpy(X).cuda())
    out = ix.query_device(torch.from_numpy(Q).cuda(), cfg.k, cfg.h, cfg.delta, cfg.seed,
                          torch.from_numpy(al).cuda(), counts=True, sums=True)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items() if k != "status" and v is not None}
    ix.close()
    del out
    torch.cuda.empty_cache()
    t_gpu = time.perf_counter() - t0
    _W.update(X=X, Q=Q, cfg=cfg, alpha=al, sums=True)
    orc.lib()
    t0 = time.perf_counter()
    mism = []
    same = 0
    with mp.get_context("fork").Pool(cores) as pool:
        for a, ref in pool.imap_unordered(_orc_one, range(q), chunksize=1):
            bad = _compare(got, ref, a, KEYS)
            if bad:
                mism.append({"query": int(a), "fields": bad})
            else:
                same += 1
    return {"config": cfg.name, "n": cfg.n, "d": cfg.d, "k": cfg.k, "h": cfg.h, "queries": q,
            "identical": same, "mismatches": mism[:20], "fields": list(KEYS),
            "gpu_call_s": round(t_gpu, 2), "oracle_s": round(time.perf_counter() - t0, 1),
            "oracle_cores": cores, "launch_path": "aknn_query_async, whole batch, graph-launched loop"}


def _orc_c5(a):
    import oracle.oracle as orc
    X, Q, cfg, al = _W["X"], _W["Q"], _W["cfg"], _W["alpha"]
    r = orc.query_br(X, Q[a:a + 1], cfg.k, cfg.h, cfg.seed, al, qids=np.array([a], np.int32),
                     want_counts=True, want_sums=False)
    return a, {k: (None if r[k] is None else r[k][0]) for k in KEYS}


def run_c5(nsample, cores):
    """Config 5 at full size: 8 shards of 1,000,000 rows on this GPU (query_multi), the
    sampled queries both inside the full 1,024-query batch and alone (qi_offset)."""
    import torch  # noqa: F401
    import oracle.oracle as orc
    import paper_1902_09465_b200 as ak
    cfg = synth.config(5)
    S = 1_000_000
    X = synth.points(cfg)
    Q = synth.queries(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    rows = np.sort(np.random.default_rng(5).permutation(cfg.q)[:nsample])
    shards = [ak.Index(X[s * S:(s + 1) * S], n_global=cfg.n, offset=s * S) for s in range(cfg.n // S)]
    t0 = time.perf_counter()
    full = ak.query_multi(shards, Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=False, sums=False)
    t_full = time.perf_counter() - t0
    alone = {}
    for a in rows:  # per-pair counts of one query at a time: n_global int32 columns
        alone[int(a)] = ak.query_multi(shards, Q[a:a + 1], cfg.k, cfg.h, cfg.delta, cfg.seed, al,
                                       counts=True, sums=False, qi_offset=int(a))
    for s in shards:
        s.close()
    _W.update(X=X, Q=Q, cfg=cfg, alpha=al)
    orc.lib()
    t0 = time.perf_counter()
    res = []
    with mp.get_context("fork").Pool(min(cores, len(rows))) as pool:
        for a, ref in pool.imap_unordered(_orc_c5, [int(r) for r in rows], chunksize=1):
            g1 = alone[a]
            bad = [k for k in ("sets", "dhat", "counts", "evals", "draws", "rounds")
                   if not np.array_equal(np.asarray(g1[k][0]), np.asarray(ref[k]))]
            badf = [k for k in ("sets", "dhat", "evals", "draws", "rounds")
                    if not np.array_equal(np.asarray(full[k][a]), np.asarray(ref[k]))]
            res.append({"query": a, "alone_mismatch": bad, "in_batch_mismatch": badf,
                        "counts_digest": int(np.bitwise_xor.reduce(
                            ref["counts"].astype(np.uint64) * np.arange(1, cfg.n + 1, dtype=np.uint64)))})
    return {"config": cfg.name, "n": cfg.n, "d": cfg.d, "k": cfg.k, "h": cfg.h, "shards": len(shards),
            "sampled_queries": [int(r) for r in rows], "results": sorted(res, key=lambda r: r["query"]),
            "identical": sum(1 for r in res if not r["alone_mismatch"] and not r["in_batch_mismatch"]),
            "full_batch_s": round(t_full, 1), "oracle_s": round(time.perf_counter() - t0, 1),
            "launch_path": "aknn_query_multi over 8 shard indices on one GPU (sharded kernels + merge)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--c5-queries", type=int, default=4)
    ap.add_argument("--nq", type=int, default=0, help="limit queries per config (smoke runs)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_parity_set.json"))
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    cores = max(1, len(os.sched_getaffinity(0)))
    recs = []
    for c in [int(x) for x in a.configs.split(",")]:
        rec = run_c5(a.c5_queries, cores) if c == 5 else run_config(c, cores, a.nq or None)
        print(json.dumps(rec), flush=True)
        recs.append(rec)
    with open(a.out, "w") as f:
        json.dump({"what": "SURVEY.md §8(d) parity set, GPU vs oracle", "records": recs}, f, indent=1)


if __name__ == "__main__":
    main()
