"""sec5.py -- the paper's §5 experiment (Figure 2) on the GPU path:
SURVEY.md §8(f) row 3.

    python bench.py --workload sec5 [--trials 20] [--c-alpha 1e-5,1e-4,1e-3,1e-2]
                                    [--sec5-schedules a1,br] [--sec5-workloads p10,p100,p1000,images]

Workloads (synth.sec5_trial): random data on p-dimensional subspaces
x = c Q y (p = 10, 100, 1000) and an image-shaped stand-in for Tiny ImageNet (config 3's
mixture recipe; the dataset is not in the container), n = 1,000 points of dimension
m = 12,288, one query per trial, k = h = 10, delta = 0.001, the §5 radius
alpha(u) = sqrt(C_alpha log(1 + (1 + log u) n / delta) / u), C_alpha swept.  As in the
paper, every trial draws a fresh point set and query, and each (workload, C_alpha)
reports the median and interquartile range over the trials of
  * recall   = |S_close ∩ Ŝ| / k (tie-aware, reading R16), S_close from the exact pass;
  * fraction = evals / (n m), the ratio of coordinate evaluations to the naive
    algorithm's (reading R14).
Both schedules run on the GPU: "a1" is the literal Algorithm 1 (the paper's own,
aknn_query_a1, one warp per query; trials in flight concurrently, one index and
stream each), "br" the batched round rule (aknn_query_ex), "br_lead<L>" the batched rule with a
close-side lead L (aknn_opts.lead, reading R24), "br_g2" the batched rule with growth factor < 2 (aknn_opts.growth = 2,
reading R25; "br_g2_lead<L>" with a lead), "br_wor" the batched rule sampling
without replacement (AKNN_FLAG_WITHOUT_REPLACEMENT, reading R23).  The exact k-NN per trial
comes from the exact tensor-core pass (aknn_exact).  The oracle is not used here.
"""
from __future__ import annotations

import concurrent.futures as cf
import json
import os
import sys
import time

import numpy as np

import synth


def _recall(X: np.ndarray, q: np.ndarray, got: np.ndarray, dk: int, k: int) -> float:
    """Tie-aware containment (reading R16): points strictly closer than the k-th exact
    distance D_(k) must all be in the set; ties at D_(k) fill the remaining slots."""
    D = ((X[got].astype(np.int64) - q.astype(np.int64)) ** 2).sum(1)
    below = int((D < dk).sum())
    tied = int((D == dk).sum())
    return (below + min(tied, max(0, k - below))) / k


def _quart(v):
    a = np.asarray(v, np.float64)
    return {"median": float(np.median(a)), "q25": float(np.percentile(a, 25)),
            "q75": float(np.percentile(a, 75))}


def run(args, dist) -> None:
    import torch
    import paper_1902_09465_b200 as ak

    torch.cuda.set_device(dist.local)
    P = synth.SEC5
    n, m, k, h, delta = P["n"], P["m"], P["k"], P["h"], P["delta"]
    trials = args.trials
    calphas = [float(c) for c in args.c_alpha.split(",")]
    scheds = [s for s in args.sec5_schedules.split(",") if s]
    works = [w for w in args.sec5_workloads.split(",") if w]
    # rank r of N runs trials r, r + N, ... (independent problems: no collective)
    mine = list(range(dist.rank, trials, dist.world))

    t_gen = time.perf_counter()
    with cf.ThreadPoolExecutor(max(1, min(16, os.cpu_count() or 1))) as pool:
        data = dict(zip([(w, t) for w in works for t in mine],
                        pool.map(lambda wt: synth.sec5_trial(*wt), [(w, t) for w in works for t in mine])))
    t_gen = time.perf_counter() - t_gen

    alphas = {c: ak.alpha_table(n, delta, m, "experimental", c) for c in calphas}
    keys = list(data)

    # phase 1 (serial): every trial's index, its exact k-NN, the batched rule for every
    # C_alpha, and the workspace Algorithm 1 needs -- so that phase 2 never allocates or
    # frees device memory (a cudaFree synchronises the whole device)
    t0 = time.perf_counter()
    ixs, dks, rows = {}, {}, []
    for wt in keys:
        w, t = wt
        X, q = data[wt]
        ix = ixs[wt] = ak.Index(X)
        _, dist2 = ix.exact(q, k)
        dks[wt] = int(dist2[0, k - 1])
        for c in calphas:
            for sname in scheds:
                if not sname.startswith("br"):
                    continue
                # "br": the batched rule; "br_lead<L>": with a close-side lead L (reading R24);
                # "br_wor": sampling without replacement (reading R23)
                # "br_g2": the growth-factor-< 2 schedule (aknn_opts.growth = 2, reading R25),
                # "br_g2_lead<L>": with a lead as well
                g2 = sname.startswith("br_g2")
                base = sname[len("br_g2"):] if g2 else sname[len("br"):]
                lead = int(base[len("_lead"):]) if base.startswith("_lead") else 1
                flags = ak.FLAG_WITHOUT_REPLACEMENT if sname == "br_wor" else 0
                t1 = time.perf_counter()
                r = ix.query(q, k, h, delta, t, alphas[c], counts=False, dhat=False, lead=lead, flags=flags,
                             growth=2 if g2 else 1)
                rows.append(dict(w=w, trial=t, c=c, s=sname, recall=_recall(X, q[0], r["sets"][0], dks[wt], k),
                                 fraction=int(r["evals"][0]) / (n * m), rounds=int(r["rounds"][0]),
                                 draws=int(r["draws"][0]), wall_s=time.perf_counter() - t1))
        if "a1" in scheds:
            ix.query(q, k, h, delta, t, alphas[calphas[0]], counts=False, dhat=False, schedule="a1", max_rounds=1)
    t_br = time.perf_counter() - t0

    # phase 2 (concurrent): Algorithm 1, one host thread per trial, each on its index's
    # own stream (one warp per query: the trials run side by side on the SMs)
    def one(wt):
        w, t = wt
        X, q = data[wt]
        out = []
        for c in calphas:
            t1 = time.perf_counter()
            r = ixs[wt].query(q, k, h, delta, t, alphas[c], counts=False, dhat=False, schedule="a1",
                              max_rounds=args.sec5_a1_max_iters)
            out.append(dict(w=w, trial=t, c=c, s="a1", recall=_recall(X, q[0], r["sets"][0], dks[wt], k),
                            fraction=int(r["evals"][0]) / (n * m), rounds=int(r["rounds"][0]),
                            draws=int(r["draws"][0]), wall_s=time.perf_counter() - t1,
                            capped=r["status"] != 0))
        print(f"sec5: {w} trial {t} done", file=sys.stderr, flush=True)
        return out

    t0 = time.perf_counter()
    if "a1" in scheds:
        with cf.ThreadPoolExecutor(max(1, min(args.sec5_threads, len(keys)))) as pool:
            rows += [r for rs in pool.map(one, keys) for r in rs]
    t_a1 = time.perf_counter() - t0
    for ix in ixs.values():
        ix.close()
    wall = t_br + t_a1
    if dist.world > 1:
        import torch.distributed as tdist
        gathered = [None] * dist.world
        tdist.all_gather_object(gathered, rows)
        rows = [r for rs in gathered for r in rs]
    if dist.rank != 0:
        return
    table = []
    for w in works:
        for c in calphas:
            for s in scheds:
                sel = [r for r in rows if r["w"] == w and r["c"] == c and r["s"] == s]
                if not sel:
                    continue
                table.append({"workload": w, "c_alpha": c, "schedule": s, "trials": len(sel),
                              "recall": _quart([r["recall"] for r in sel]),
                              "fraction": _quart([r["fraction"] for r in sel]),
                              "rounds_median": float(np.median([r["rounds"] for r in sel])),
                              "capped": int(sum(bool(r.get("capped")) for r in sel)),
                              "wall_s_median": float(np.median([r["wall_s"] for r in sel]))})
    print(json.dumps({
        "metric": "recall and fraction of naive coordinate evaluations vs C_alpha (P:349-359, Figure 2)",
        "workload": "sec5_figure2", "n_gpus": dist.world, "data": "synthetic (synth.sec5_trial; DESIGN.md §14)",
        "config": {"n": n, "m": m, "k": k, "h": h, "delta": delta, "trials": trials,
                   "c_alpha": calphas, "schedules": scheds, "workloads": works,
                   "alpha": "P:349 alpha(u) = sqrt(C_alpha log(1 + (1 + log u) n / delta) / u)",
                   "seed": "Philox key = trial index"},
        "wall_s": wall, "br_phase_s": t_br, "a1_phase_s": t_a1, "generate_s": t_gen,
        "table": table}), flush=True)
