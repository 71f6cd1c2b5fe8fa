"""GPU parity (-m gpu): the CUDA path through the C-ABI vs the CPU oracle.

Bar: integer outputs (sets, per-pair counts T_i, per-pair sums
S_i, draws, evals, rounds) bit-exact; the fp64 estimates d_hat to 0 ulp
(np.array_equal on float64).  Inputs are seeded synthetic data (synth/)."""
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


def _assert_parity(got, ref, keys=KEYS, rows=None):
    for k in keys:
        g = got[k] if rows is None else got[k][rows]
        assert g.shape == ref[k].shape, (k, g.shape, ref[k].shape)
        if not np.array_equal(g, ref[k]):
            bad = np.argwhere(np.atleast_1d(g != ref[k]))[:5]
            raise AssertionError(f"{k} differs at {bad.tolist()}")


def _run_both(ak, X, Q, k, h, seed, alpha, **kw):
    ix = ak.Index(X)
    got = ix.query(Q, k, h, 0.05, seed, alpha, counts=True, sums=True, **kw)
    ix.close()
    ref = orc.query_br(X, Q, k, h, seed, alpha, want_sums=True,
                       max_rounds=kw.get("max_rounds", 0))
    return got, ref


def test_config1_full_bit_exact(ak):
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    got, ref = _run_both(ak, X, Q, cfg.k, cfg.h, cfg.seed, al)
    _assert_parity(got, ref)
    assert sorted(got["sets"][0].tolist()) == planted.tolist()


CASES = [
    # (name, n, d, q, k, h, alpha kind, c_alpha, seed, data kind)
    ("ragged_n_d", 1237, 100, 5, 3, 4, "theory", 0, 1, "mixture"),
    ("d_not16", 777, 33, 7, 5, 5, "exp", 0.05, 2, "mixture"),
    ("many_rounds_mixed_levels", 3001, 256, 6, 4, 6, "exp", 0.02, 3, "mixture"),
    ("h0_lucb", 900, 64, 4, 6, 0, "exp", 0.1, 4, "mixture"),
    ("uniform_hard", 4099, 128, 3, 10, 10, "theory", 0, 5, "uniform"),
    ("n_above_select_cap", 20011, 96, 3, 7, 9, "exp", 0.05, 6, "mixture"),
    ("tiny_n", 5, 16, 4, 2, 2, "theory", 0, 7, "uniform"),
    ("d2", 300, 2, 3, 3, 3, "theory", 0, 8, "uniform"),
    ("d3", 300, 3, 3, 3, 3, "exp", 0.1, 9, "uniform"),
    ("large_k", 5000, 48, 2, 300, 200, "exp", 0.05, 10, "mixture"),
    ("row_staged_d5000", 1500, 5000, 2, 5, 5, "theory", 0, 11, "mixture"),
    ("row_staged_exp", 3000, 8192, 2, 4, 4, "exp", 0.3, 12, "mixture"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_small_instances_bit_exact(ak, case):
    name, n, d, q, k, h, kind, c, seed, data = case
    X, Q = synth.small_instance(100 + seed, n, d, q=q, kind=data)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, c)
    got, ref = _run_both(ak, X, Q, k, h, 0xDEADBEEF00000000 + seed, al)
    _assert_parity(got, ref)


def test_d1_exact_after_init(ak):
    rng = np.random.default_rng(3)
    X = rng.integers(0, 256, (500, 1), dtype=np.uint8)
    Q = rng.integers(0, 256, (4, 1), dtype=np.uint8)
    al = orc.alpha_theory(500, 0.05, 1)
    got, ref = _run_both(ak, X, Q, 3, 3, 0, al)
    _assert_parity(got, ref)
    assert np.all(got["rounds"] == 1)


def test_max_rounds_partial_state(ak):
    X, Q = synth.small_instance(55, 2000, 200, q=4)
    al = orc.alpha_theory(2000, 0.05, 200)
    got, ref = _run_both(ak, X, Q, 5, 5, 3, al, max_rounds=3)
    assert got["status"] == ak.AKNN_EMAXROUNDS and ref["status"] == orc.EMAXROUNDS
    _assert_parity(got, ref)


def test_qi_offset_selects_rng_stream(ak):
    X, Q = synth.small_instance(56, 800, 64, q=6)
    al = orc.alpha_experimental(800, 0.05, 64, 0.1)
    ix = ak.Index(X)
    full = ix.query(Q, 4, 4, 0.05, 11, al, sums=True)
    part = ix.query(Q[3:], 4, 4, 0.05, 11, al, sums=True, qi_offset=3)
    ix.close()
    for k in ("sets", "counts", "sums", "rounds"):
        assert np.array_equal(full[k][3:], part[k])


@pytest.mark.parametrize("i,n,q", [(2, 6000, 8), (3, 1500, 3), (4, 20000, 3), (5, 8000, 4)])
def test_reduced_configs_bit_exact(ak, i, n, q):
    """Configs 2-5 at a prefix of their rows and queries (oracle finishes in seconds)."""
    cfg = synth.config(i)
    X = synth.points(cfg, 0, n)
    Q = synth.queries(cfg)[:q]
    al = orc.alpha_theory(n, cfg.delta, cfg.d)
    got, ref = _run_both(ak, X, Q, cfg.k, cfg.h, cfg.seed, al)
    _assert_parity(got, ref)


def test_config2_full_size_sampled_queries(ak):
    """Config 2 at its BASELINE size (the bench workload, same launch path: device API,
    all 1000 queries in one call); the oracle recomputes 3 sampled queries in full."""
    import torch
    cfg = synth.config(2)
    X = synth.points(cfg)
    Q = synth.queries(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    ix = ak.Index(torch.from_numpy(X).cuda())
    out = ix.query_device(torch.from_numpy(Q).cuda(), cfg.k, cfg.h, cfg.delta, cfg.seed, al,
                          counts=True, sums=True)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items() if k != "status" and v is not None}
    ix.close()
    rows = np.random.default_rng(2).choice(cfg.q, 3, replace=False)
    ref = orc.query_br(X, Q[rows], cfg.k, cfg.h, cfg.seed, al, qids=rows, want_sums=True)
    _assert_parity(got, ref, rows=rows)


@pytest.mark.parametrize("i,nsample", [(3, 1), (4, 2), (5, 1)])
def test_full_size_configs_sampled_queries(ak, i, nsample):
    """Configs 3 and 4 at their BASELINE sizes, config 5 at one GPU's shard (its first
    1,000,000 rows: the N=1 bench workload), through the bench launch path (device API,
    the whole query batch in one call, graph-launched loop); the oracle recomputes
    `nsample` seeded queries of the batch in full (sets, d_hat, per-pair T and S,
    draws, evals, rounds)."""
    import torch
    cfg = synth.config(i)
    X = synth.points(cfg, 0, 1_000_000) if cfg.shards > 1 else synth.points(cfg)
    if cfg.shards > 1:
        cfg = synth.config(i, n=X.shape[0])
    Q = synth.queries(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    ix = ak.Index(torch.from_numpy(X).cuda())
    rows = np.random.default_rng(i).choice(cfg.q, nsample, replace=False)
    out = ix.query_device(torch.from_numpy(Q).cuda(), cfg.k, cfg.h, cfg.delta, cfg.seed, al,
                          counts=True, sums=True)
    torch.cuda.synchronize()
    got = {k: v[torch.as_tensor(rows).cuda()].cpu().numpy()
           for k, v in out.items() if k != "status" and v is not None}
    ix.close()
    del out
    ref = orc.query_br(X, Q[rows], cfg.k, cfg.h, cfg.seed, al, qids=rows, want_sums=True)
    _assert_parity(got, ref)


def test_device_api_equals_host_api(ak):
    import torch
    X, Q = synth.small_instance(77, 3000, 120, q=9)
    al = orc.alpha_experimental(3000, 0.05, 120, 0.05)
    ix = ak.Index(X)
    host = ix.query(Q, 5, 5, 0.05, 21, al, counts=True, sums=True)
    dev = ix.query_device(torch.from_numpy(Q).cuda(), 5, 5, 0.05, 21, al, counts=True, sums=True)
    torch.cuda.synchronize()
    for k in KEYS:
        assert np.array_equal(host[k], dev[k].cpu().numpy()), k
    # determinism: a second run is byte-identical
    again = ix.query(Q, 5, 5, 0.05, 21, al, counts=True, sums=True)
    for k in KEYS:
        assert np.array_equal(host[k], again[k]), k
    ix.close()


def test_null_alpha_uses_footnote2_table(ak):
    X, Q = synth.small_instance(78, 700, 40, q=2)
    ix = ak.Index(X)
    a = ix.query(Q, 3, 3, 0.05, 1, None, sums=True)
    b = ix.query(Q, 3, 3, 0.05, 1, orc.alpha_theory(700, 0.05, 40), sums=True)
    ix.close()
    for k in KEYS[:-1]:
        if a[k] is not None:
            assert np.array_equal(a[k], b[k]), k


def test_invalid_arguments_rejected(ak):
    X, Q = synth.small_instance(79, 50, 8, q=1)
    ix = ak.Index(X)
    al = orc.alpha_theory(50, 0.05, 8)
    for kw in (dict(k=25, h=25), dict(k=0, h=1), dict(k=1, h=-1)):
        with pytest.raises(ak.AknnError):
            ix.query(Q, kw["k"], kw["h"], 0.05, 0, al)
    with pytest.raises(ak.AknnError):
        ix.query(Q, 2, 2, 1.5, 0, al)
    with pytest.raises(ak.AknnError):
        ix.query(np.zeros((1, 9), np.uint8), 2, 2, 0.05, 0, al)
    ix.close()


# --------------------------------------------------------------------------- exact pass
@pytest.mark.parametrize("n,d,q,k,lo,hi", [(1000, 256, 1, 5, 0, 256), (5003, 100, 70, 17, 0, 256),
                                           (3000, 64, 9, 50, 0, 2), (129, 784, 130, 128, 0, 256)])
def test_exact_pass_vs_bruteforce(ak, n, d, q, k, lo, hi):
    """aknn_exact == oracle brute force, ties (values in {0,1}) by smaller id."""
    rng = np.random.default_rng(n + d)
    X = rng.integers(lo, hi, (n, d), dtype=np.uint8)
    Q = rng.integers(lo, hi, (q, d), dtype=np.uint8)
    ix = ak.Index(X)
    idx, dist = ix.exact(Q, k)
    ix.close()
    ridx, rdist = orc.bruteforce(X, Q, k)
    assert np.array_equal(idx, ridx)
    assert np.array_equal(dist, rdist)


@pytest.mark.parametrize("max_rounds", [0, 3])
def test_graph_loop_equals_host_loop(ak, max_rounds):
    """The device-driven loop (CUDA graph with a conditional WHILE node, timing off) and
    the host-driven loop (timing on: per-launch events) give identical bytes, also when
    the round cap stops the batch (EMAXROUNDS)."""
    X, Q = synth.small_instance(91, 2500, 140, q=7)
    al = orc.alpha_experimental(2500, 0.05, 140, 0.05)
    ix = ak.Index(X)
    a = ix.query(Q, 6, 4, 0.05, 5, al, counts=True, sums=True, max_rounds=max_rounds)
    b = ix.query(Q, 6, 4, 0.05, 5, al, counts=True, sums=True, max_rounds=max_rounds, timing=True)
    sa = ix.stats()
    c = ix.query(Q, 6, 4, 0.05, 5, al, counts=True, sums=True, max_rounds=max_rounds)  # cached graph
    sc = ix.stats()
    ix.close()
    assert a["status"] == b["status"] == c["status"]
    for k in KEYS:
        assert np.array_equal(a[k], b[k]) and np.array_equal(a[k], c[k]), k
    assert sa["rounds"] == sc["rounds"] and sa["query_rounds"] == sc["query_rounds"]
    assert sa["blocked_query_rounds"] == sc["blocked_query_rounds"]
    ref = orc.query_br(X, Q, 6, 4, 5, al, want_sums=True, max_rounds=max_rounds)
    _assert_parity(a, ref)


@pytest.mark.parametrize("n,d,q,k,h", [(20011, 96, 3, 7, 9), (30000, 64, 4, 40, 40), (700, 32, 3, 3, 3)])
def test_pivot_select_equals_radix_select(ak, n, d, q, k, h):
    """The one-pass pivot rank split and the multi-pass radix select (forced with
    AKNN_FLAG_RADIX_SELECT) decide every round identically; both equal the oracle."""
    X, Q = synth.small_instance(n + 1, n, d, q=q)
    al = orc.alpha_experimental(n, 0.05, d, 0.05)
    ix = ak.Index(X)
    a = ix.query(Q, k, h, 0.05, 9, al, counts=True, sums=True)
    b = ix.query(Q, k, h, 0.05, 9, al, counts=True, sums=True, flags=ak.FLAG_RADIX_SELECT)
    ix.close()
    for key in KEYS:
        assert np.array_equal(a[key], b[key]), key
    _assert_parity(a, orc.query_br(X, Q, k, h, 9, al, want_sums=True))


def test_sharded_radix_flag_equals_pivot(ak):
    X, Q = synth.small_instance(5, 12000, 48, q=3)
    al = orc.alpha_experimental(12000, 0.05, 48, 0.05)
    sh = [ak.Index(X[a:b], n_global=12000, offset=a) for a, b in ((0, 5000), (5000, 12000))]
    a = ak.query_multi(sh, Q, 8, 8, 0.05, 4, al, counts=True, sums=True)
    b = ak.query_multi(sh, Q, 8, 8, 0.05, 4, al, counts=True, sums=True, flags=ak.FLAG_RADIX_SELECT)
    for s in sh:
        s.close()
    for key in KEYS:
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("n,d,q,k,h,kind", [(3001, 256, 6, 4, 6, "theory"), (1237, 100, 131, 3, 4, "theory"),
                                            (777, 33, 7, 5, 5, "exp"), (5, 16, 4, 2, 2, "theory"),
                                            (2000, 784, 3, 10, 10, "theory")])
def test_exact_fallback_tensor_cores_equals_rows(ak, n, d, q, k, h, kind):
    """Exact fallbacks computed by the tcgen05 tile pass (default) and by per-pair
    row streams (AKNN_FLAG_EXACT_ROWS) give identical bytes; both equal the oracle.  q = 131
    spans two 128-query tiles; n = 1237 and 3001 leave ragged point tiles."""
    X, Q = synth.small_instance(n + d, n, d, q=q)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, 0.05)
    ix = ak.Index(X)
    a = ix.query(Q, k, h, 0.05, 21, al, counts=True, sums=True, flags=ak.FLAG_EXACT_MMA_ALL)
    sa = ix.stats()
    b = ix.query(Q, k, h, 0.05, 21, al, counts=True, sums=True, flags=ak.FLAG_EXACT_ROWS)
    c = ix.query(Q, k, h, 0.05, 21, al, counts=True, sums=True)  # dense tiles only on the MMA
    ix.close()
    for key in KEYS:
        assert np.array_equal(a[key], b[key]), key
        assert np.array_equal(a[key], c[key]), key
    if n > 100:
        assert sa["exact_fallbacks"] > 0  # the tile pass was exercised
    _assert_parity(a, orc.query_br(X, Q, k, h, 21, al, want_sums=True))


@pytest.mark.parametrize("n,d,q,k,h,kind", [(3001, 256, 6, 4, 6, "theory"), (1237, 100, 70, 3, 4, "theory"),
                                            (4099, 128, 3, 10, 10, "exp"), (5, 16, 4, 2, 2, "theory"),
                                            (2000, 784, 35, 10, 10, "theory"), (700, 5000, 3, 4, 4, "theory")])
def test_tiled_advance_equals_lists(ak, n, d, q, k, h, kind):
    """Level gathers of dense tiles from shared memory (default) and through the work
    lists (AKNN_FLAG_NO_TILES) give identical bytes; both equal the oracle.  Ragged n
    and q leave partial tiles; d = 5000 takes the smallest tile shape."""
    X, Q = synth.small_instance(n + 3 * d, n, d, q=q)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, 0.05)
    ix = ak.Index(X)
    a = ix.query(Q, k, h, 0.05, 33, al, counts=True, sums=True)
    b = ix.query(Q, k, h, 0.05, 33, al, counts=True, sums=True, flags=ak.FLAG_NO_TILES)
    c = ix.query(Q, k, h, 0.05, 33, al, counts=True, sums=True,
                 flags=ak.FLAG_NO_TILES | ak.FLAG_EXACT_ROWS)
    ix.close()
    for key in KEYS:
        assert np.array_equal(a[key], b[key]), key
        assert np.array_equal(a[key], c[key]), key
    _assert_parity(a, orc.query_br(X, Q, k, h, 33, al, want_sums=True))


def test_sharded_tiles_equal_lists(ak):
    X, Q = synth.small_instance(77, 9000, 200, q=5)
    al = orc.alpha_theory(9000, 0.05, 200)
    sh = [ak.Index(X[a:b], n_global=9000, offset=a) for a, b in ((0, 4001), (4001, 9000))]
    a = ak.query_multi(sh, Q, 8, 8, 0.05, 4, al, counts=True, sums=True)
    b = ak.query_multi(sh, Q, 8, 8, 0.05, 4, al, counts=True, sums=True, flags=ak.FLAG_NO_TILES)
    for s in sh:
        s.close()
    for key in KEYS:
        assert np.array_equal(a[key], b[key]), key
    _assert_parity(a, orc.query_br(X, Q, 8, 8, 4, al, want_sums=True))


def test_async_call_defers_stats(ak):
    """aknn_query_async on the graph path returns without waiting; its statistics are
    completed by aknn_get_stats or by the next call, and equal the host API's."""
    import torch
    X, Q = synth.small_instance(404, 3000, 160, q=300)  # several 128-query exact tiles
    al = orc.alpha_theory(3000, 0.05, 160)
    ix = ak.Index(X)
    Qd = torch.from_numpy(Q).cuda()
    a1 = ix.query_device(Qd, 5, 5, 0.05, 1, al)
    a2 = ix.query_device(Qd, 5, 5, 0.05, 2, al)  # finishes the first call's statistics
    torch.cuda.synchronize()
    s2 = ix.stats()
    h2 = ix.query(Q, 5, 5, 0.05, 2, al, counts=False)
    hs2 = ix.stats()
    h1 = ix.query(Q, 5, 5, 0.05, 1, al, counts=False)
    ix.close()
    for key in ("sets", "dhat", "evals", "draws", "rounds"):
        assert np.array_equal(a1[key].cpu().numpy(), h1[key]), key
        assert np.array_equal(a2[key].cpu().numpy(), h2[key]), key
    for key in ("draws", "rounds", "exact_fallbacks", "philox_blocks", "query_rounds", "kernel_launches"):
        assert s2[key] == hs2[key], key


# --------------------------------------------------------------- query-independent draws
@pytest.mark.parametrize("n,d,q,k,h,kind", [(3001, 256, 40, 4, 6, "theory"), (1237, 100, 70, 3, 4, "exp"),
                                            (2000, 784, 35, 10, 10, "theory"), (700, 5000, 3, 4, 4, "theory")])
def test_shared_draws_bit_exact(ak, n, d, q, k, h, kind):
    """AKNN_FLAG_SHARED_DRAWS == the oracle with the shared counter word,
    through the tiles and through the lists."""
    X, Q = synth.small_instance(n + 5 * d, n, d, q=q)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, 0.05)
    ix = ak.Index(X)
    a = ix.query(Q, k, h, 0.05, 41, al, counts=True, sums=True, flags=ak.FLAG_SHARED_DRAWS)
    b = ix.query(Q, k, h, 0.05, 41, al, counts=True, sums=True,
                 flags=ak.FLAG_SHARED_DRAWS | ak.FLAG_NO_TILES)
    ix.close()
    for key in KEYS:
        assert np.array_equal(a[key], b[key]), key
    _assert_parity(a, orc.query_br(X, Q, k, h, 41, al, want_sums=True, shared_draws=True))


def test_shared_draws_config1_and_reduced_config2(ak):
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    ix = ak.Index(X)
    got = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True,
                   flags=ak.FLAG_SHARED_DRAWS)
    ix.close()
    _assert_parity(got, orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, shared_draws=True))
    assert sorted(got["sets"][0].tolist()) == planted.tolist()
    cfg = synth.config(2)
    X = synth.points(cfg, 0, 6000)
    Q = synth.queries(cfg)[:40]
    al = orc.alpha_theory(6000, cfg.delta, cfg.d)
    ix = ak.Index(X)
    got = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True,
                   flags=ak.FLAG_SHARED_DRAWS)
    ix.close()
    _assert_parity(got, orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, shared_draws=True))


@pytest.mark.parametrize("n,d,q,k,h,kind", [(20011, 100, 130, 5, 5, "theory"), (9000, 784, 64, 10, 10, "theory"),
                                            (6001, 48, 257, 4, 4, "exp")])
def test_shared_draws_level_mma(ak, n, d, q, k, h, kind):
    """Shared draws with the round's dominant level as tensor-core GEMMs (k_level_mma,
    default) == the per-pair gathers (AKNN_FLAG_NO_LEVEL_MMA) == the oracle.  Ragged n
    and q leave partial 128 x 128 tiles; the GEMM path must actually have run."""
    X, Q = synth.small_instance(n + 7 * d, n, d, q=q)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, 0.05)
    ix = ak.Index(X)
    a = ix.query(Q, k, h, 0.05, 43, al, counts=True, sums=True, flags=ak.FLAG_SHARED_DRAWS)
    sa = ix.stats()
    b = ix.query(Q, k, h, 0.05, 43, al, counts=True, sums=True,
                 flags=ak.FLAG_SHARED_DRAWS | ak.FLAG_NO_LEVEL_MMA)
    ix.close()
    assert sa["level_mma_tiles"] > 0
    for key in KEYS:
        assert np.array_equal(a[key], b[key]), key
    rows = np.arange(0, q, max(1, q // 6))
    ref = orc.query_br(X, Q[rows], k, h, 43, al, want_sums=True, shared_draws=True)
    _assert_parity(a, ref, rows=rows)


@pytest.mark.parametrize("groups", ["0", "2", "4", "5", "8", "10", "24"])
def test_grouped_tiles_wide_rows(ak, groups, monkeypatch):
    """Rows wider than 8 KB (C3-like, d = 12,288 and 9,000): the grouped tile kernel
    (AKNN_TILE_GROUPS = 2, 4, 5 (two query rows per group), 8, 10, 24 thread groups sharing
    the column's point rows) and the
    classic one (0) agree with the oracle bit for bit, including ragged q and n."""
    monkeypatch.setenv("AKNN_TILE_GROUPS", groups)
    monkeypatch.setenv("AKNN_TILE_F", "0.25")  # make most tiles dense at small levels too
    for (n, d, q, seed) in ((1203, 12288, 7, 41), (700, 9000, 5, 42)):
        X, Q = synth.small_instance(seed, n, d, q=q)
        al = orc.alpha_experimental(n, 0.05, d, 0.3)
        got, ref = _run_both(ak, X, Q, 4, 4, seed, al)
        _assert_parity(got, ref)


def test_grouped_tiles_tight_rows(ak, monkeypatch):
    """The grouped kernel with rows at the pitch (AKNN_TILE_TIGHT = 1: 2 groups x 1 query
    row + 16 point rows) against the oracle."""
    monkeypatch.setenv("AKNN_TILE_GROUPS", "2")
    monkeypatch.setenv("AKNN_TILE_TIGHT", "1")
    monkeypatch.setenv("AKNN_TILE_F", "0.25")
    for (n, d, q, seed) in ((1203, 12288, 7, 43), (777, 9000, 5, 44)):
        X, Q = synth.small_instance(seed, n, d, q=q)
        al = orc.alpha_experimental(n, 0.05, d, 0.3)
        got, ref = _run_both(ak, X, Q, 4, 4, seed, al)
        _assert_parity(got, ref)


@pytest.mark.parametrize("db", ["0", "1"])
def test_grouped_tiles_two_groups(ak, db, monkeypatch):
    """Two groups per CTA, with (AKNN_TILE_DB = 1) and without double-buffered query rows,
    over several point columns per CTA, against the oracle."""
    monkeypatch.setenv("AKNN_TILE_GROUPS", "2")
    monkeypatch.setenv("AKNN_TILE_DB", db)
    monkeypatch.setenv("AKNN_TILE_F", "0.25")
    X, Q = synth.small_instance(45, 4000, 12288, q=9)
    al = orc.alpha_experimental(4000, 0.05, 12288, 0.3)
    got, ref = _run_both(ak, X, Q, 4, 4, 45, al)
    _assert_parity(got, ref)


def test_grouped_tiles_eight_groups(ak, monkeypatch):
    """Eight 2-warp groups with rows at the pitch (AKNN_TILE_GROUPS = 8) against the oracle."""
    monkeypatch.setenv("AKNN_TILE_GROUPS", "8")
    monkeypatch.setenv("AKNN_TILE_F", "0.25")
    for (n, d, q, seed) in ((4000, 12288, 9, 46), (777, 9000, 5, 47)):
        X, Q = synth.small_instance(seed, n, d, q=q)
        al = orc.alpha_experimental(n, 0.05, d, 0.3)
        got, ref = _run_both(ak, X, Q, 4, 4, seed, al)
        _assert_parity(got, ref)


def test_grouped_tiles_shared_draws(ak, monkeypatch):
    """Query-independent draws through the grouped tiles (rows > 8 KB) against the oracle's
    shared-draw mode."""
    monkeypatch.setenv("AKNN_TILE_F", "0.25")
    X, Q = synth.small_instance(48, 2100, 12288, q=6)
    al = orc.alpha_experimental(2100, 0.05, 12288, 0.3)
    ix = ak.Index(X)
    got = ix.query(Q, 4, 4, 0.05, 48, al, counts=True, sums=True, flags=ak.FLAG_SHARED_DRAWS)
    ix.close()
    ref = orc.query_br(X, Q, 4, 4, 48, al, want_sums=True, shared_draws=True)
    _assert_parity(got, ref)


@pytest.mark.parametrize("zs", ["4", "64", "1024"])
def test_z_tiles(ak, zs, monkeypatch):
    """|x - q| tiles (k_advance_tiles_z: each pair's row |x_p - q| materialised once, one
    byte gather per draw) for the tiles whose pairs draw >= AKNN_TILE_ZS each, the rest in
    the grouped kernel: bit-exact against the oracle over mixed levels, ragged n and q,
    several point columns per CTA, and rows that are not a multiple of 128 bytes (d = 9,000)."""
    monkeypatch.setenv("AKNN_TILE_ZS", zs)
    monkeypatch.setenv("AKNN_TILE_F", "0.25")
    for (n, d, q, seed) in ((1203, 12288, 7, 51), (700, 9000, 5, 52), (4000, 12288, 9, 53)):
        X, Q = synth.small_instance(seed, n, d, q=q)
        al = orc.alpha_experimental(n, 0.05, d, 0.3)
        got, ref = _run_both(ak, X, Q, 4, 4, seed, al)
        _assert_parity(got, ref)


def test_z_tiles_shared_draws(ak, monkeypatch):
    """Query-independent draws through the |x - q| tiles against the oracle's shared-draw mode."""
    monkeypatch.setenv("AKNN_TILE_ZS", "4")
    monkeypatch.setenv("AKNN_TILE_F", "0.25")
    X, Q = synth.small_instance(54, 2100, 12288, q=6)
    al = orc.alpha_experimental(2100, 0.05, 12288, 0.3)
    ix = ak.Index(X)
    got = ix.query(Q, 4, 4, 0.05, 54, al, counts=True, sums=True, flags=ak.FLAG_SHARED_DRAWS)
    ix.close()
    ref = orc.query_br(X, Q, 4, 4, 54, al, want_sums=True, shared_draws=True)
    _assert_parity(got, ref)


@pytest.mark.parametrize("qg", ["0", "32", "65536"])
def test_qg_tiles(ak, qg, monkeypatch):
    """The grouped kernel's QG variant (the query byte of each draw gathered from global
    memory, no query-row copies, super tiles of several query rows) for the dense tiles
    whose pairs draw < AKNN_TILE_QG each (65,536: every dense tile; 0: none), the rest in
    the plain grouped kernel: bit-exact against the oracle over mixed levels, ragged n and
    q (rows past q, non-dense rows inside a super tile), several columns per CTA."""
    monkeypatch.setenv("AKNN_TILE_QG", qg)
    monkeypatch.setenv("AKNN_TILE_F", "0.25")
    for (n, d, q, seed) in ((1203, 12288, 7, 61), (700, 9000, 21, 62), (4000, 12288, 9, 63)):
        X, Q = synth.small_instance(seed, n, d, q=q)
        al = orc.alpha_experimental(n, 0.05, d, 0.3)
        got, ref = _run_both(ak, X, Q, 4, 4, seed, al)
        _assert_parity(got, ref)
