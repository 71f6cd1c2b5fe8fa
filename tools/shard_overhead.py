"""Sharded-round overhead on ONE GPU: the same C5-shaped batch over the
same points as one index vs W shard indices driven in lockstep by aknn_query_multi
(k_select_local_pivot + k_merge per round instead of k_select_pivot; the transport is a
shared receive buffer instead of ncclAllGather).  Results must be identical; prints the
wall time of each (host API, inputs resident).  Not a bench line: a diagnostic."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_1902_09465_b200 as ak  # noqa: E402

n, q, W = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000, 256, 2
cfg = synth.config(5, n=n, q=q)
X = synth.points(synth.config(5), 0, n)
Q = synth.queries(cfg)
al = ak.alpha_table(n, cfg.delta, cfg.d, "theory")
one = ak.Index(X)
cuts = [i * n // W for i in range(W + 1)]
sh = [ak.Index(X[a:b], n_global=n, offset=a) for a, b in zip(cuts[:-1], cuts[1:])]
out = {}
for name, fn in (("one_index", lambda: one.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=False)),
                 (f"{W}_shards", lambda: ak.query_multi(sh, Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=False))):
    fn()
    t0 = time.perf_counter()
    r = fn()
    out[name] = (time.perf_counter() - t0, r)
a, b = out["one_index"][1], out[f"{W}_shards"][1]
same = all(np.array_equal(a[k], b[k]) for k in ("sets", "dhat", "evals", "draws", "rounds"))
print(json.dumps({"n": n, "q": q, "d": cfg.d, "k": cfg.k, "h": cfg.h, "shards": W,
                  "one_index_s": out["one_index"][0], "sharded_s": out[f"{W}_shards"][0],
                  "identical": same, "rounds_max": int(a["rounds"].max())}))
