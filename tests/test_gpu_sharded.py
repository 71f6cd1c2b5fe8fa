"""GPU parity of the point-sharded round (-m gpu).

The shards of one point set live on one device and are driven in lockstep by
aknn_query_multi: the same select/summary/merge kernels as the NCCL path, with
the transport replaced by a shared receive buffer (one GPU per run here; see
B200_PROFILING.md on not emulating ranks with kernels that wait on each other).
Bar: bit-identical to the oracle on the unsharded set (sets, d_hat to 0 ulp,
per-pair counts/sums, draws, evals, rounds)."""
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


def _shards(ak, X, cuts):
    n = X.shape[0]
    bounds = [0, *cuts, n]
    return [ak.Index(X[a:b], n_global=n, offset=a) for a, b in zip(bounds[:-1], bounds[1:])]


def _check(got, ref):
    for k in KEYS:
        assert got[k].shape == ref[k].shape, k
        if not np.array_equal(got[k], ref[k]):
            bad = np.argwhere(np.atleast_1d(got[k] != ref[k]))[:5]
            raise AssertionError(f"{k} differs at {bad.tolist()}")


CASES = [
    # name, n, d, q, k, h, alpha, c, cuts (shard boundaries)
    ("two_even", 2000, 64, 4, 5, 5, "exp", 0.05, [1000]),
    ("three_ragged", 3001, 100, 5, 4, 6, "theory", 0, [777, 2100]),
    ("four_uneven_h0", 2500, 48, 3, 6, 0, "exp", 0.1, [100, 1300, 1400]),
    ("eight_shards", 4000, 32, 3, 10, 10, "exp", 0.05, [500 * i for i in range(1, 8)]),
    ("one_shard_equals_unsharded", 1500, 80, 4, 5, 5, "theory", 0, []),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_multi_shard_bit_exact_vs_oracle(ak, case):
    name, n, d, q, k, h, kind, c, cuts = case
    X, Q = synth.small_instance(300 + n, n, d, q=q)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, c)
    shards = _shards(ak, X, cuts)
    got = ak.query_multi(shards, Q, k, h, 0.05, 77, al, counts=True, sums=True)
    for s in shards:
        s.close()
    ref = orc.query_br(X, Q, k, h, 77, al, want_sums=True)
    _check(got, ref)


def test_multi_shard_max_rounds(ak):
    X, Q = synth.small_instance(311, 1800, 120, q=3)
    al = orc.alpha_theory(1800, 0.05, 120)
    shards = _shards(ak, X, [600, 1200])
    got = ak.query_multi(shards, Q, 5, 5, 0.05, 3, al, counts=True, sums=True, max_rounds=4)
    for s in shards:
        s.close()
    ref = orc.query_br(X, Q, 5, 5, 3, al, want_sums=True, max_rounds=4)
    assert got["status"] == ak.AKNN_EMAXROUNDS
    _check(got, ref)


def test_config5_prefix_sharded_like_the_bench(ak):
    """Config 5's recipe (k = h = 100, delta = 0.01) on a 16,000-row prefix split into 8
    shards of 2,000 rows, 3 queries, against the oracle on the unsharded prefix."""
    cfg = synth.config(5)
    n = 16_000
    X = synth.points(cfg, 0, n)
    Q = synth.queries(cfg)[:3]
    al = orc.alpha_theory(n, cfg.delta, cfg.d)
    shards = _shards(ak, X, [2000 * i for i in range(1, 8)])
    got = ak.query_multi(shards, Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True)
    for s in shards:
        s.close()
    ref = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True)
    _check(got, ref)


def test_multi_rejects_bad_tilings(ak):
    X, Q = synth.small_instance(312, 1000, 16, q=1)
    al = orc.alpha_theory(1000, 0.05, 16)
    a = ak.Index(X[:500], n_global=1000, offset=0)
    b = ak.Index(X[600:], n_global=1000, offset=600)
    with pytest.raises(ak.AknnError):
        ak.query_multi([a, b], Q, 3, 3, 0.05, 0, al)
    c = ak.Index(X[500:], n_global=1000, offset=500)
    with pytest.raises(ak.AknnError):  # k + h must be < every shard's n_local
        ak.query_multi([a, c], Q, 300, 300, 0.05, 0, al)
    for s in (a, b, c):
        s.close()
