"""GPU parity of the close-side lead (aknn_opts.lead; DESIGN.md
reading R24) against the oracle's lead mode: sets, per-pair counts and sums, draws,
evals and rounds bit-exact, d_hat to 0 ulp -- through the dense tiles, the work lists,
the row-stream exact fallbacks, point shards, and combined with the other stream
variants (shared draws, sampling without replacement)."""
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


def _eq(got, ref):
    for k in KEYS:
        assert got[k].shape == ref[k].shape, (k, got[k].shape, ref[k].shape)
        if not np.array_equal(got[k], ref[k]):
            bad = np.argwhere(np.atleast_1d(got[k] != ref[k]))[:5]
            raise AssertionError(f"{k} differs at {bad.tolist()}")


CASES = [
    # (name, n, d, q, k, h, alpha kind, c_alpha, lead)
    ("ragged_l2", 1237, 100, 5, 3, 4, "exp", 0.05, 2),
    ("mixed_l3", 3001, 256, 6, 4, 6, "exp", 0.02, 3),
    ("tiles_d784_l3", 2000, 784, 35, 10, 10, "exp", 0.1, 3),
    ("theory_l4", 1500, 128, 4, 5, 5, "theory", 0, 4),
    ("h0_l5", 900, 64, 4, 6, 0, "exp", 0.1, 5),
    ("staged_l2", 1500, 5000, 2, 5, 5, "exp", 0.3, 2),
    ("tiny_l8", 5, 16, 4, 2, 2, "theory", 0, 8),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_lead_bit_exact_three_paths(ak, case):
    name, n, d, q, k, h, kind, c, lead = case
    X, Q = synth.small_instance(1300 + n + d, n, d, q=q)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, c)
    seed = 0xBEEF + lead
    ix = ak.Index(X)
    try:
        a = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, lead=lead)
        b = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, lead=lead, flags=ak.FLAG_NO_TILES)
        c2 = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, lead=lead,
                      flags=ak.FLAG_NO_TILES | ak.FLAG_EXACT_ROWS)
        t = ix.query(Q, k, h, 0.05, seed, al, counts=True, sums=True, lead=lead, timing=True)
    finally:
        ix.close()
    ref = orc.query_br(X, Q, k, h, seed, al, want_sums=True, lead=lead)
    for got in (a, b, c2, t):
        _eq(got, ref)


def test_lead_config1_planted(ak):
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_experimental(cfg.n, cfg.delta, cfg.d, 0.1)
    ix = ak.Index(X)
    got = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True, lead=3)
    base = ix.query(Q, cfg.k, cfg.h, cfg.delta, cfg.seed, al, counts=True, sums=True)
    ix.close()
    _eq(got, orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, want_sums=True, lead=3))
    assert sorted(got["sets"][0].tolist()) == planted.tolist()
    assert got["evals"][0] < base["evals"][0]


@pytest.mark.parametrize("variant", ["shared", "wor"])
def test_lead_with_stream_variants(ak, variant):
    X, Q = synth.small_instance(1351, 2500, 200, q=40)
    al = orc.alpha_experimental(2500, 0.05, 200, 0.05)
    ix = ak.Index(X)
    flags = ak.FLAG_SHARED_DRAWS if variant == "shared" else ak.FLAG_WITHOUT_REPLACEMENT
    got = ix.query(Q, 6, 6, 0.05, 3, al, counts=True, sums=True, lead=3, flags=flags)
    ix.close()
    ref = orc.query_br(X, Q, 6, 6, 3, al, want_sums=True, lead=3, shared_draws=variant == "shared",
                       without_replacement=variant == "wor")
    _eq(got, ref)


def test_lead_point_shards(ak):
    X, Q = synth.small_instance(1352, 3001, 100, q=5)
    al = orc.alpha_experimental(3001, 0.05, 100, 0.05)
    sh = [ak.Index(X[a:b], n_global=3001, offset=a) for a, b in ((0, 777), (777, 2100), (2100, 3001))]
    try:
        got = ak.query_multi(sh, Q, 4, 6, 0.05, 77, al, counts=True, sums=True, lead=3)
    finally:
        for s in sh:
            s.close()
    _eq(got, orc.query_br(X, Q, 4, 6, 77, al, want_sums=True, lead=3))


def test_lead_out_of_range_rejected(ak):
    X, Q = synth.small_instance(1353, 200, 16, q=2)
    ix = ak.Index(X)
    try:
        with pytest.raises(ak.AknnError):
            ix.query(Q, 3, 3, 0.05, 0, orc.alpha_theory(200, 0.05, 16), lead=9)
    finally:
        ix.close()


@pytest.mark.parametrize("max_rounds", [1, 2, 4])
def test_lead_round_cap_partial_state(ak, max_rounds):
    """A round cap stops after whole rounds (every lead pass of the last round done):
    the partial state equals the oracle's, on the graph loop and the host loop."""
    X, Q = synth.small_instance(1360, 1500, 96, q=6)
    al = orc.alpha_experimental(1500, 0.05, 96, 0.05)
    ix = ak.Index(X)
    try:
        g = ix.query(Q, 5, 5, 0.05, 8, al, counts=True, sums=True, lead=3, max_rounds=max_rounds)
        t = ix.query(Q, 5, 5, 0.05, 8, al, counts=True, sums=True, lead=3, max_rounds=max_rounds,
                     timing=True)
    finally:
        ix.close()
    ref = orc.query_br(X, Q, 5, 5, 8, al, want_sums=True, lead=3, max_rounds=max_rounds)
    _eq(g, ref)
    _eq(t, ref)
