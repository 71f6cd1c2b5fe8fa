"""Pins of the oracle's growth schedule (reading R25):
R6 takes an arm from T samples to next(T) samples, next(T) the smallest integer of the
grid G_m = {(m + r) 2^j / m : j >= 0, 0 <= r < m} above T.  m = 1 is the batched
rule's doubling; m = 2 grows by 3/2 and 4/3 alternately (sqrt 2 per level on average),
m = 4 by at most 5/4 -- growth factors < 2 that cut the doubling overshoot.

Pinned by hand-written count sequences, the closed-form ratio bound, m = 1 being the
batched rule byte for byte, and by what no schedule can change: every arm sums the first
T of its own (cuRAND-pinned) sample stream, exact arms hold the brute-force distance,
and the returned set contains the exact k nearest neighbours."""
import numpy as np
import pytest

import oracle.oracle as orc
import synth

SEQ = {
    1: [1, 2, 4, 8, 16, 32, 64, 128, 256],
    2: [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128],
    4: [1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 14, 16, 20, 24, 28, 32, 40, 48, 56, 64],
}


@pytest.mark.parametrize("m", [1, 2, 4])
def test_next_count_sequences(m):
    seq = [1]
    while len(seq) < len(SEQ[m]):
        seq.append(orc.next_count(seq[-1], m))
    assert seq == SEQ[m]


@pytest.mark.parametrize("m,bound", [(2, 1.5), (4, 1.25)])
def test_next_count_ratio_and_powers_of_two(m, bound):
    """next(T)/T <= 3/2 (m = 2, T >= 2) and 5/4 (m = 4, T >= 4); every power of two is
    a count, so an advance never straddles two sample levels b of the Draw stream."""
    lo = 2 if m == 2 else 4
    for T in [v for v in range(lo, 5000)]:
        n = orc.next_count(T, m)
        assert n > T and n / T <= bound + 1e-12
        p = 1 << (T.bit_length() - 1)  # the power of two at or below T
        assert n <= 2 * p  # [T, next(T)) lies inside [p, 2p): one level b
    for j in range(20):
        assert orc.next_count((1 << j) - 1, m) == (1 << j) or (1 << j) - 1 < lo


def test_growth_one_is_the_batched_rule():
    X, Q = synth.small_instance(801, 500, 96, q=3)
    al = orc.alpha_experimental(500, 0.05, 96, 0.1)
    a = orc.query_br(X, Q, 4, 4, 2, al, want_sums=True)
    b = orc.query_br(X, Q, 4, 4, 2, al, want_sums=True, growth=1)
    for key in ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("m", [2, 4])
def test_growth_counts_and_sums_are_the_arm_streams(m):
    X, Q = synth.small_instance(802, 150, 40, q=2)
    n, d = X.shape
    seed = 11
    al = orc.alpha_experimental(n, 0.05, d, 0.05)
    r = orc.query_br(X, Q, 3, 3, seed, al, want_sums=True, growth=m)
    grid = set(SEQ[m]) | {orc.next_count(t, m) for t in range(1, d)}
    D = ((X[None].astype(np.int64) - Q[:, None].astype(np.int64)) ** 2).sum(2)
    for a in range(2):
        for i in range(n):
            T = int(r["counts"][a, i])
            if T == d:
                assert r["sums"][a, i] == D[a, i]
            else:
                assert T in grid and T < d  # a sampled count of the schedule
                js = [orc.draw_index(seed, a, i, t, d) for t in range(T)]
                want = int(((X[i, js].astype(np.int64) - Q[a, js].astype(np.int64)) ** 2).sum())
                assert r["sums"][a, i] == want


@pytest.mark.parametrize("m", [2, 4])
def test_growth_keeps_the_knn_guarantee(m):
    fails = 0
    for s in range(30):
        X, Q = synth.small_instance(810 + s, 200, 48, q=2)
        al = orc.alpha_theory(200, 0.05, 48)
        r = orc.query_br(X, Q, 5, 5, s, al, growth=m)
        idx, _ = orc.bruteforce(X, Q, 5)
        for a in range(2):
            fails += not set(idx[a].tolist()) <= set(r["sets"][a].tolist())
    assert fails <= 3  # delta = 0.05 over 60 queries (Theorem 1); in practice 0


def test_growth_planted_set_and_accounting():
    """C1 returns its 10 planted points under every schedule; draws = the sampled counts
    (sum of T over sampled arms plus the last sampled count of every exact arm), and
    evals = draws + d per exact arm, which bounds draws by the arms' exact-trigger counts."""
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_experimental(cfg.n, cfg.delta, cfg.d, 0.1)
    for m in (1, 2, 4):
        r = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, growth=m)
        assert sorted(r["sets"][0].tolist()) == planted.tolist()
        T = r["counts"][0]
        nexact = int((T == cfg.d).sum())
        assert r["evals"][0] == r["draws"][0] + cfg.d * nexact
        assert r["draws"][0] >= int(T[T < cfg.d].sum())
