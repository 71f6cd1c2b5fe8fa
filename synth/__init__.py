"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is the ONLY code shared by the oracle side (tests, cpu_baseline)
and the product side (bench.py, smoke): it produces input bytes and the
config parameters and contains none of the method's arithmetic.

Recipes (BASELINE.json ``configs``):
  * numpy ``default_rng`` (PCG64).  "round" = ``np.rint`` (ties to even),
    then ``clip(0, 255)``.  Cluster labels are i.i.d. uniform; queries are
    fresh draws from the same mixture, not members of X.
  * Rows are generated in fixed chunks of ``CHUNK`` rows, chunk c drawing
    from ``SeedSequence(seed).spawn(...)[2 + c]``, so any row range (a shard,
    a prefix for a reduced-n test) is reproducible on its own.
  * Mixture noise is drawn as float32 standard normals times sigma, added to
    float64 centres uniform on [0, 255).
Stand-ins: configs 2 and 3 copy only the SHAPES of MNIST and Tiny ImageNet
(P:349); neither dataset is in the container and no item of either is used.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

CHUNK = 50_000


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    q: int
    k: int
    h: int
    delta: float
    data_seed: int
    kind: str            # "planted" | "mixture" | "uniform"
    centres: int = 0
    sigma: float = 0.0
    seed: int = 0        # Philox key for the method's draws
    shards: int = 1


CONFIGS = [
    Config("c1_tiny_planted", n=1_000, d=256, q=1, k=5, h=5, delta=0.05, data_seed=0,
           kind="planted"),
    Config("c2_mnist_shaped", n=60_000, d=784, q=1_000, k=10, h=10, delta=0.05, data_seed=2,
           kind="mixture", centres=10, sigma=40.0),
    Config("c3_tinyimagenet_shaped", n=100_000, d=12_288, q=256, k=10, h=10, delta=0.05,
           data_seed=3, kind="mixture", centres=200, sigma=30.0),
    Config("c4_hard_uniform", n=1_000_000, d=1_024, q=128, k=50, h=50, delta=0.05,
           data_seed=4, kind="uniform"),
    Config("c5_sharded", n=8_000_000, d=768, q=1_024, k=100, h=100, delta=0.01, data_seed=5,
           kind="mixture", centres=1_000, sigma=35.0, shards=8),
]


def config(i: int, **over) -> Config:
    """Config i (1-based, as in BASELINE.json), optionally with n/q/k/h overridden."""
    return dataclasses.replace(CONFIGS[i - 1], **over)


def _mixture_rows(rng: np.random.Generator, centres: np.ndarray, sigma: float, m: int):
    lab = rng.integers(0, centres.shape[0], m)
    noise = rng.standard_normal((m, centres.shape[1]), dtype=np.float32)
    rows = centres[lab].astype(np.float32) + noise * np.float32(sigma)
    return np.clip(np.rint(rows), 0, 255).astype(np.uint8)


def _seqs(cfg: Config, nchunks: int):
    return np.random.SeedSequence(cfg.data_seed).spawn(2 + nchunks)


def points(cfg: Config, row0: int = 0, row1: Optional[int] = None) -> np.ndarray:
    """Rows [row0, row1) of the config's point set X, uint8 [rows, d]."""
    row1 = cfg.n if row1 is None else row1
    if cfg.kind == "planted":
        return planted(cfg)[0][row0:row1]
    nchunks = (max(row1, cfg.n) + CHUNK - 1) // CHUNK
    seqs = _seqs(cfg, nchunks)
    centres = None
    if cfg.kind == "mixture":
        centres = np.random.default_rng(seqs[0]).uniform(0.0, 255.0, (cfg.centres, cfg.d))
    out = np.empty((row1 - row0, cfg.d), np.uint8)
    for c in range(row0 // CHUNK, (row1 + CHUNK - 1) // CHUNK):
        lo, hi = c * CHUNK, min((c + 1) * CHUNK, cfg.n)
        rng = np.random.default_rng(seqs[2 + c])
        if cfg.kind == "mixture":
            blk = _mixture_rows(rng, centres, cfg.sigma, hi - lo)
        else:
            blk = rng.integers(0, 256, (hi - lo, cfg.d), dtype=np.uint8)
        a, b = max(lo, row0), min(hi, row1)
        out[a - row0:b - row0] = blk[a - lo:b - lo]
    return out


def queries(cfg: Config) -> np.ndarray:
    """The config's query rows, uint8 [q, d]."""
    if cfg.kind == "planted":
        return planted(cfg)[1]
    seqs = _seqs(cfg, 0)
    rng = np.random.default_rng(seqs[1])
    if cfg.kind == "mixture":
        centres = np.random.default_rng(seqs[0]).uniform(0.0, 255.0, (cfg.centres, cfg.d))
        return _mixture_rows(rng, centres, cfg.sigma, cfg.q)
    return rng.integers(0, 256, (cfg.q, cfg.d), dtype=np.uint8)


def planted(cfg: Config):
    """Config 1: q ~ U(uint8^d); 10 planted rows clip(q + U{-8..8}); the rest uniform.

    Returns (X, Q, planted_indices)."""
    rng = np.random.default_rng(cfg.data_seed)
    qv = rng.integers(0, 256, cfg.d)
    pos = rng.permutation(cfg.n)[:10]
    X = rng.integers(0, 256, (cfg.n, cfg.d)).astype(np.uint8)
    X[pos] = np.clip(qv[None, :] + rng.integers(-8, 9, (10, cfg.d)), 0, 255).astype(np.uint8)
    return X, qv.astype(np.uint8)[None, :], np.sort(pos)


def small_instance(seed: int, n: int, d: int, q: int = 1, kind: str = "mixture",
                   centres: int = 4, sigma: float = 30.0):
    """Tiny seeded instances for oracle and parity tests (same recipes, small shapes)."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        X = rng.integers(0, 256, (n, d), dtype=np.uint8)
        Q = rng.integers(0, 256, (q, d), dtype=np.uint8)
        return X, Q
    cen = rng.uniform(0.0, 255.0, (centres, d))
    return _mixture_rows(rng, cen, sigma, n), _mixture_rows(rng, cen, sigma, q)


# ---------------------------------------------------------------------------
# §5 workloads.  Each trial is an independent
# problem: n points and one query drawn from the same generator.
SEC5 = dict(n=1_000, m=12_288, k=10, h=10, delta=0.001, trials=20, seed=1902)
SEC5_WORKLOADS = ("p10", "p100", "p1000", "images")


def subspace_trial(p: int, trial: int, n: int = SEC5["n"], m: int = SEC5["m"],
                   seed: int = SEC5["seed"]):
    """x = c Q y, Q in R^{m x p} i.i.d. Gaussian with unit-norm columns, y uniform
    on the unit sphere of R^p, c the largest scalar with ||x||_inf <= 1/2 over the
    generated set (the n points and the query).  Stored as uint8 u = rint(255 (x + 1/2))
    (reading R22: one sample (u_a - u_b)^2 / 65025 ~ (x_a - x_b)^2, the
    paper's [0, 1] sample range).  Returns (X uint8 [n, m], q uint8 [1, m])."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, p, trial]))
    Qm = rng.standard_normal((m, p))
    Qm /= np.linalg.norm(Qm, axis=0, keepdims=True)
    Y = rng.standard_normal((n + 1, p))
    Y /= np.linalg.norm(Y, axis=1, keepdims=True)
    Xr = Y @ Qm.T
    Xr *= 0.5 / np.abs(Xr).max()
    U = np.clip(np.rint((Xr + 0.5) * 255.0), 0, 255).astype(np.uint8)
    return np.ascontiguousarray(U[:n]), np.ascontiguousarray(U[n:])


def images_trial(trial: int, n: int = SEC5["n"], seed: int = SEC5["seed"]):
    """Stand-in for P:349's Tiny ImageNet trials (the dataset is not in the container):
    n + 1 rows of config 3's mixture recipe (its 200 centres, sigma 30, d = 12,288), the
    last one the query.  Returns (X uint8 [n, d], q uint8 [1, d])."""
    c3 = config(3)
    centres = np.random.default_rng(_seqs(c3, 0)[0]).uniform(0.0, 255.0, (c3.centres, c3.d))
    rows = _mixture_rows(np.random.default_rng(np.random.SeedSequence([seed, 0, trial])), centres, c3.sigma, n + 1)
    return np.ascontiguousarray(rows[:n]), np.ascontiguousarray(rows[n:])


def sec5_trial(workload: str, trial: int, **kw):
    """One §5 trial of `workload` in SEC5_WORKLOADS."""
    if workload == "images":
        return images_trial(trial, **{k: v for k, v in kw.items() if k in ("n", "seed")})
    return subspace_trial(int(workload[1:]), trial, **kw)
