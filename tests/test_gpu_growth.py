"""GPU parity (-m gpu) of the growth-factor schedule (DESIGN.md
reading R25; aknn_opts.growth = 2: counts 1, 2, 3, 4, 6, 8, 12, ...) against the
oracle's growth mode: sets, d_hat, per-pair counts and sums, draws, evals and rounds
bit-exact.  Growth 2 runs the list path (k_advance with the generic level advance) and
the exact fallbacks on the tensor cores or as row streams; it composes with the
close-side lead, point shards and the host-driven loop."""
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
        if not np.array_equal(got[k], ref[k]):
            bad = np.argwhere(np.atleast_1d(got[k] != ref[k]))[:5]
            raise AssertionError(f"{k} differs at {bad.tolist()}")


CASES = [
    # name, n, d, q, k, h, alpha kind, c_alpha, seed
    ("small_theory", 1237, 100, 5, 3, 4, "theory", 0, 1),
    ("d_not16_exp", 777, 33, 7, 5, 5, "exp", 0.05, 2),
    ("many_levels", 3001, 256, 6, 4, 6, "exp", 0.02, 3),
    ("h0", 900, 64, 4, 6, 0, "exp", 0.1, 4),
    ("wide_rows", 1500, 5000, 2, 5, 5, "theory", 0, 5),
    ("d2", 300, 2, 3, 3, 3, "theory", 0, 6),
    ("d3", 300, 3, 3, 3, 3, "exp", 0.1, 7),
    ("d5", 400, 5, 3, 3, 3, "theory", 0, 8),
    ("large_k", 5000, 48, 2, 100, 60, "exp", 0.05, 9),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_growth2_bit_exact(ak, case):
    _, n, d, q, k, h, kind, c, seed = case
    X, Q = synth.small_instance(300 + seed, n, d, q=q)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, c)
    ix = ak.Index(X)
    got = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, growth=2)
    rows = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, growth=2, flags=ak.FLAG_EXACT_ROWS,
                    timing=True)
    ix.close()
    ref = orc.query_br(X, Q, k, h, seed, al, want_sums=True, growth=2)
    _eq(got, ref)
    _eq(rows, ref)


def test_growth2_config1_and_lead(ak):
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_experimental(cfg.n, cfg.delta, cfg.d, 0.1)
    ix = ak.Index(X)
    for lead in (1, 3):
        got = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True, growth=2, lead=lead)
        ref = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, growth=2, lead=lead)
        _eq(got, ref)
        assert sorted(got["sets"][0].tolist()) == planted.tolist()
    ix.close()


def test_growth2_reduced_config2_and_max_rounds(ak):
    cfg = synth.config(2)
    X = synth.points(cfg, 0, 6000)
    Q = synth.queries(cfg)[:6]
    al = orc.alpha_theory(6000, cfg.delta, cfg.d)
    ix = ak.Index(X)
    got = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True, growth=2)
    cap = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True, growth=2, max_rounds=5,
                   batch_queries=4)
    ix.close()
    _eq(got, orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, growth=2))
    assert cap["status"] == ak.AKNN_EMAXROUNDS
    _eq(cap, orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, growth=2, max_rounds=5))


def test_growth2_sharded(ak):
    X, Q = synth.small_instance(333, 4000, 96, q=5)
    al = orc.alpha_theory(4000, 0.05, 96)
    shards = [ak.Index(X[a:b], n_global=4000, offset=a) for a, b in ((0, 1500), (1500, 4000))]
    got = ak.query_multi(shards, Q, 4, 4, 0.05, 3, al, sums=True, growth=2)
    for s in shards:
        s.close()
    _eq(got, orc.query_br(X, Q, 4, 4, 3, al, want_sums=True, growth=2))


def test_growth_one_is_default_and_invalid_combinations(ak):
    X, Q = synth.small_instance(334, 800, 64, q=3)
    al = orc.alpha_experimental(800, 0.05, 64, 0.1)
    ix = ak.Index(X)
    a = ix.query(Q, 3, 3, 0.05, 1, al, sums=True)
    b = ix.query(Q, 3, 3, 0.05, 1, al, sums=True, growth=1)
    _eq(a, b)
    for kw in (dict(growth=3), dict(growth=-1), dict(growth=2, flags=ak.FLAG_SHARED_DRAWS),
               dict(growth=2, flags=ak.FLAG_WITHOUT_REPLACEMENT)):
        with pytest.raises(ak.AknnError):
            ix.query(Q, 3, 3, 0.05, 1, al, **kw)
    ix.close()
