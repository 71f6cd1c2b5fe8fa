"""GPU parity of sampling WITHOUT replacement (AKNN_FLAG_WITHOUT_REPLACEMENT; footnote 1
to P:120; reading R23) against the oracle's
without_replacement mode: sets, per-pair counts and sums, draws, evals and rounds
bit-exact, d_hat to 0 ulp -- through every path that draws coordinates (init, list
levels, lane-group levels, row-staged levels, dense tiles, exact fallbacks on the tensor
cores and as row streams, point shards, the literal Algorithm 1)."""
import numpy as np
import pytest

import oracle.oracle as orc
import synth

pytestmark = pytest.mark.gpu

KEYS = ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds")


@pytest.fixture(scope="module")
def ak():
    import torch
    torch.cuda.set_device(0)
    import paper_1902_09465_b200 as m
    return m


def _eq(got, ref, keys=KEYS):
    for k in keys:
        assert got[k].shape == ref[k].shape, (k, got[k].shape, ref[k].shape)
        if not np.array_equal(got[k], ref[k]):
            bad = np.argwhere(np.atleast_1d(got[k] != ref[k]))[:5]
            raise AssertionError(f"{k} differs at {bad.tolist()}")


def _alpha(kind, n, d, c):
    return orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, c)


CASES = [
    # (name, n, d, q, k, h, alpha kind, c_alpha, data kind)
    ("ragged", 1237, 100, 5, 3, 4, "theory", 0, "mixture"),
    ("d_not16", 777, 33, 7, 5, 5, "exp", 0.05, "mixture"),
    ("mixed_levels", 3001, 256, 6, 4, 6, "exp", 0.02, "mixture"),
    ("tiles_d784", 2000, 784, 35, 10, 10, "theory", 0, "mixture"),
    ("uniform_hard", 4099, 128, 3, 10, 10, "theory", 0, "uniform"),
    ("tiny", 5, 16, 4, 2, 2, "theory", 0, "uniform"),
    ("d2", 300, 2, 3, 3, 3, "theory", 0, "uniform"),
    ("d3", 300, 3, 3, 3, 3, "exp", 0.1, "uniform"),
    ("row_staged", 1500, 5000, 2, 5, 5, "theory", 0, "mixture"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_wor_bit_exact_three_paths(ak, case):
    """Default (tiles + tensor-core fallbacks), work lists only, and work lists with
    row-stream fallbacks: identical bytes, equal to the oracle."""
    name, n, d, q, k, h, kind, c, data = case
    X, Q = synth.small_instance(900 + n + d, n, d, q=q, kind=data)
    al = _alpha(kind, n, d, c)
    seed = 0xC0FFEE00 + d
    ix = ak.Index(X)
    try:
        F = ak.FLAG_WITHOUT_REPLACEMENT
        a = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, flags=F)
        b = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, flags=F | ak.FLAG_NO_TILES)
        c2 = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True,
                      flags=F | ak.FLAG_NO_TILES | ak.FLAG_EXACT_ROWS)
        plain = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True)
    finally:
        ix.close()
    ref = orc.query_br(X, Q, k, h, seed, al, want_sums=True, without_replacement=True)
    _eq(a, ref)
    _eq(b, ref)
    _eq(c2, ref)
    # the closed form of reading R23: evals = sum of the final counts <= n d
    assert np.array_equal(a["evals"], a["counts"].astype(np.int64).sum(1))
    sampled = (a["counts"] < d) & (plain["counts"] < d) & (a["counts"] > 1)
    if sampled.any():  # a different stream (arms that went exact agree by construction)
        assert not np.array_equal(plain["sums"][sampled], a["sums"][sampled])


def test_wor_config1_planted(ak):
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    ix = ak.Index(X)
    got = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True,
                   flags=ak.FLAG_WITHOUT_REPLACEMENT)
    ix.close()
    _eq(got, orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, without_replacement=True))
    assert sorted(got["sets"][0].tolist()) == planted.tolist()


def test_wor_reduced_config2(ak):
    cfg = synth.config(2)
    X, Q = synth.points(cfg, 0, 6000), synth.queries(cfg)[:8]
    al = orc.alpha_theory(6000, cfg.delta, cfg.d)
    ix = ak.Index(X)
    got = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True,
                   flags=ak.FLAG_WITHOUT_REPLACEMENT)
    ix.close()
    _eq(got, orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, without_replacement=True))


def test_wor_point_shards(ak):
    X, Q = synth.small_instance(911, 3001, 100, q=5)
    al = orc.alpha_theory(3001, 0.05, 100)
    sh = [ak.Index(X[a:b], n_global=3001, offset=a) for a, b in ((0, 777), (777, 2100), (2100, 3001))]
    try:
        got = ak.query_multi(sh, Q, 4, 6, 0.05, 77, al, counts=True, sums=True,
                             flags=ak.FLAG_WITHOUT_REPLACEMENT)
    finally:
        for s in sh:
            s.close()
    _eq(got, orc.query_br(X, Q, 4, 6, 77, al, want_sums=True, without_replacement=True))


A1_CASES = [("a1_mixture", 333, 40, 3, 3, 4, 0.05), ("a1_uniform", 257, 32, 2, 5, 5, 0.2),
            ("a1_walk_to_d", 60, 12, 2, 3, 3, 2.0)]


@pytest.mark.parametrize("case", A1_CASES, ids=[c[0] for c in A1_CASES])
def test_wor_algorithm1(ak, case):
    name, n, d, q, k, h, c = case
    X, Q = synth.small_instance(920 + n, n, d, q=q, kind="uniform" if "uniform" in name or "walk" in name else "mixture")
    al = orc.alpha_experimental(n, 0.05, d, c)
    ix = ak.Index(X)
    got = ix.query(Q, k, h, 0.05, 5, al, counts=True, sums=True, schedule="a1",
                   flags=ak.FLAG_WITHOUT_REPLACEMENT)
    ix.close()
    for a in range(q):
        r = orc.query_a1(X, Q[a], k, h, 5, al, qi=a, without_replacement=True)
        assert r["status"] == 0
        assert np.array_equal(got["sets"][a], r["set"])
        assert np.array_equal(got["counts"][a], r["counts"])
        assert np.array_equal(got["sums"][a], r["sums"])
        assert (got["evals"][a], got["draws"][a], got["rounds"][a]) == (r["evals"], r["draws"], r["iters"])


def test_wor_with_shared_draws_rejected(ak):
    X, Q = synth.small_instance(930, 200, 16, q=2)
    ix = ak.Index(X)
    try:
        with pytest.raises(ak.AknnError):
            ix.query(Q, 3, 3, 0.05, 0, orc.alpha_theory(200, 0.05, 16),
                     flags=ak.FLAG_WITHOUT_REPLACEMENT | ak.FLAG_SHARED_DRAWS)
    finally:
        ix.close()
