"""Pins of the oracle's sampling WITHOUT replacement (footnote 1 to P:120; SURVEY.md
§8(f) row 4; reading R23).

The permutation is new arithmetic with no library counterpart, so it is pinned by what
the mathematics fixes: pi is a bijection of [0, d) for every key (exhaustive), the
Feistel network is a bijection of its 2*hb-bit domain, pi(t) is uniform over keys, a
full permutation's sampled sum IS the exact distance (checked by brute force inside
Algorithm 1 and here), and the evaluation accounting of R23 has a closed form.
"""
import numpy as np
import pytest

import oracle.oracle as orc
import synth

DS = [1, 2, 3, 5, 16, 17, 40, 255, 256, 257, 768, 784, 1000, 1024, 4097, 12288]


@pytest.mark.parametrize("d", DS)
def test_permutation_is_a_bijection(d):
    for seed, qi, i in [(0, 0, 0), (7, 3, 11), (2**63 + 5, 2**32 - 1, 12345)]:
        p = orc.wor_perm(seed, qi, i, d)
        assert np.array_equal(np.sort(p), np.arange(d, dtype=np.uint32))


def test_radix_domain_is_tight():
    # a = ceil(sqrt d), b = ceil(d / a): d <= a b < d + a, so cycle walking is rare
    for d in DS + [2, 7, 99, 33025]:
        a, b = orc.wor_radix(d)
        assert (a - 1) ** 2 < d <= a * a and d <= a * b < d + a


@pytest.mark.parametrize("d", [2, 6, 17, 40, 784, 1000, 12288])
def test_feistel_is_a_bijection_of_its_domain(d):  # before the cycle walk and rotation
    a, b = orc.wor_radix(d)
    keys = orc.wor_keys(3, 1, d)
    img = sorted(orc.feistel(keys, a, b, x) for x in range(a * b))
    assert img == list(range(a * b))


def test_keys_are_the_philox_block_of_the_reserved_level():
    # counter (0, i, qi, 0x80000000): the Philox routine pinned against cuRAND
    seed, qi, i = 0x1234_5678_9ABC_DEF0, 9, 77
    w = orc.philox4x32_10([0, i, qi, 0x80000000], [seed & 0xFFFFFFFF, seed >> 32])
    assert np.array_equal(orc.wor_keys(seed, qi, i), np.asarray(w, np.uint32))


def test_position_is_uniform_over_keys():
    # pi(t) for fixed t over 20,000 arms: chi-square against uniform on [0, d)
    d, trials = 40, 20_000
    for t in (0, 1, 39):
        hist = np.zeros(d)
        for i in range(trials):
            hist[orc.wor_index(orc.wor_keys(5, 0, i), d, t)] += 1
        chi2 = ((hist - trials / d) ** 2 / (trials / d)).sum()
        assert chi2 < 90, chi2  # 39 dof: p ~ 1e-5


def test_first_two_positions_are_distinct_and_pairwise_uniform():
    d, trials = 17, 60_000
    cnt = np.zeros((d, d))
    for i in range(trials):
        p = orc.wor_perm(11, 2, i, d)
        cnt[p[0], p[1]] += 1
    assert np.all(np.diag(cnt) == 0)
    off = cnt[~np.eye(d, dtype=bool)]
    exp = trials / (d * (d - 1))
    assert ((off - exp) ** 2 / exp).sum() < 360  # 271 dof: p ~ 2e-4


def test_running_mean_is_unbiased():
    rng = np.random.default_rng(0)
    d, T = 100, 10
    v = rng.integers(0, 65026, d).astype(np.float64)
    means = [v[orc.wor_perm(1, 0, i, d)[:T]].mean() for i in range(4000)]
    se = v.std() * np.sqrt((d - T) / (d - 1) / T) / np.sqrt(4000)  # finite-population s.e.
    assert abs(np.mean(means) - v.mean()) < 5 * se


def test_a1_full_permutation_sums_are_exact():
    """A1 without replacement: an arm that reaches T = d has summed every coordinate
    once; the oracle checks its running sum against the brute-force distance before the
    P:176 step (EINTERNAL otherwise), and charges nothing extra (evals = draws)."""
    X, Q = synth.small_instance(801, 60, 12, q=1, kind="uniform")
    al = orc.alpha_experimental(60, 0.05, 12, 2.0)  # wide radii: many arms walk to d
    r = orc.query_a1(X, Q[0], 3, 3, 5, al, without_replacement=True)
    assert r["status"] == 0
    full = r["counts"] == 12
    assert full.sum() >= 5
    D = ((X.astype(np.int64) - Q[0].astype(np.int64)) ** 2).sum(1)
    assert np.array_equal(r["sums"][full], D[full])
    assert r["evals"] == r["draws"] == int(r["counts"].sum())


def test_a1_sums_are_prefix_sums_of_the_permutation():
    X, Q = synth.small_instance(802, 40, 30, q=1)
    al = orc.alpha_experimental(40, 0.05, 30, 0.3)
    r = orc.query_a1(X, Q[0], 2, 2, 9, al, without_replacement=True)
    for i in range(40):
        T = int(r["counts"][i])
        p = orc.wor_perm(9, 0, i, 30)[:T]
        assert r["sums"][i] == int(((X[i, p].astype(np.int64) - Q[0, p].astype(np.int64)) ** 2).sum())


def test_br_accounting_and_prefix_sums():
    """BR without replacement: sampled arms hold the prefix sums of their permutation;
    an exact fallback is charged only the d - T coordinates not yet drawn, so
    evals = sum of the final counts <= n d (sample fraction <= 1)."""
    X, Q = synth.small_instance(803, 120, 50, q=3)
    n, d = X.shape
    al = orc.alpha_theory(n, 0.05, d)
    r = orc.query_br(X, Q, 3, 3, 4, al, want_sums=True, without_replacement=True)
    for a in range(3):
        cnt = r["counts"][a]
        assert r["evals"][a] == int(cnt.sum()) <= n * d
        for i in range(n):
            if cnt[i] < d:
                p = orc.wor_perm(4, a, i, d)[:cnt[i]]
                assert r["sums"][a, i] == int(((X[i, p].astype(np.int64) - Q[a, p].astype(np.int64)) ** 2).sum())
    D = ((X[None].astype(np.int64) - Q[:, None].astype(np.int64)) ** 2).sum(2)
    ex = r["counts"] == d
    assert ex.any() and np.array_equal(r["sums"][ex], D[ex])


def test_br_planted_set_and_knn_containment():
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    r = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, without_replacement=True)
    assert sorted(r["sets"][0].tolist()) == planted.tolist()
    X, Q = synth.small_instance(804, 300, 64, q=8)
    al = orc.alpha_theory(300, 0.05, 64)
    r = orc.query_br(X, Q, 5, 5, 1, al, without_replacement=True)
    idx, _ = orc.bruteforce(X, Q, 5)
    for a in range(8):
        assert set(idx[a].tolist()) <= set(r["sets"][a].tolist())


def test_wor_differs_from_with_replacement_and_is_schedule_independent():
    """The same per-arm streams under both schedules (A1 and BR draw pi(t) for the t-th
    sample): an arm's A1 sum at T equals the BR prefix sum of the same length."""
    X, Q = synth.small_instance(805, 200, 256, q=1)
    al = orc.alpha_experimental(200, 0.05, 256, 0.01)
    a = orc.query_a1(X, Q[0], 2, 2, 3, al, without_replacement=True)
    b = orc.query_br(X, Q, 2, 2, 3, al, without_replacement=False, want_sums=True)
    c = orc.query_br(X, Q, 2, 2, 3, al, without_replacement=True, want_sums=True)
    sampled = c["counts"][0] < 256
    assert sampled.sum() > 100
    assert not np.array_equal(b["sums"][0][sampled], c["sums"][0][sampled])
    same = 0
    for i in range(200):
        T = int(a["counts"][i])
        if T == int(c["counts"][0, i]) and T < 256:
            assert a["sums"][i] == c["sums"][0, i]
            same += 1
    assert same > 10
