"""Hand-built pins of the oracle's round rule and of
Algorithm 1's b2 choice (Eq. 4), with every expected value written by hand.

Every state below is chosen so that all fp64 quantities are exact dyadic numbers
(d_hat = S / (65025 T) = v/16 exactly because S = 65025 T v / 16 is an integer,
alpha[T] = a/16), so the equality cases of R3-R5 are real equalities and each
strict inequality of the rules is exercised on both sides:

    R3: d1 = argmax_C U, d2 = argmin_F L, ties to the smaller id
    R4: stop iff A <= B
    R5: blockers = {C: U > B} u {F: L < A} u {M: alpha > alpha_d2} minus exact arms
        (P:148-153, P:166-169 batched)

A plausible slip (a `>=` for `>`, a dropped exact-arm exclusion, a rank-order
instead of id tie-break) changes one of the hand-written expectations.
"""
import numpy as np
import pytest

import oracle.oracle as orc
import synth  # noqa: F401  (inputs only)

D = 256  # dimension of the hand-built states; T = 256 means exact


def _state(arms):
    """arms: list of (T, v) with d_hat = v/16 -> S, T arrays."""
    T = np.array([t for t, _ in arms], np.int32)
    S = np.array([65025 * t * v // 16 for t, v in arms], np.int64)
    assert all(65025 * t * v % 16 == 0 for t, v in arms)
    return S, T


def _alpha():
    """alpha[16] = 4/16, alpha[32] = 2/16, alpha[64] = 1/16; alpha[D] = 0 (exact)."""
    a = np.full(D + 1, 100.0)
    a[0] = 0.0
    a[16], a[32], a[64] = 4 / 16, 2 / 16, 1 / 16
    a[D] = 0.0
    return a


# (T, v): id -> U = v + a, L = v - a in units of 1/16 (a = 4, 2, 1 for T = 16, 32, 64; 0 exact)
BLOCKER_ARMS = [
    (64, 4),   # 0  C  U=5 == B        -> not a blocker (U > B is strict)
    (32, 5),   # 1  C  U=7 > B         -> blocker; d1 (A = 7)
    (D, 6),    # 2  C  exact, U=6 > B  -> excluded (exact arms never advance)
    (16, 6),   # 3  M  alpha 4 > 2     -> blocker
    (32, 6),   # 4  M  alpha 2 == 2    -> not a blocker (alpha > alpha_d2 is strict)
    (32, 7),   # 5  F  L=5 = B         -> d2 (tie with id 10 -> smaller id); L < A -> blocker
    (64, 8),   # 6  F  L=7 == A        -> not a blocker (L < A is strict)
    (32, 8),   # 7  F  L=6 < A         -> blocker
    (D, 6),    # 8  F  exact, L=6 < A  -> excluded; ranks after M by the id tie-break
    (64, 9),   # 9  F  L=8 > A         -> not a blocker
    (32, 7),   # 10 F  L=5 = B, L < A  -> blocker (loses the d2 tie to id 5)
]


def test_blocker_set_every_branch():
    S, T = _state(BLOCKER_ARMS)
    r = orc.round_step(S, T, D, 3, 2, _alpha())
    # R2: order by (d_hat, id): v = 4,5,6,6,6,6(id 8),7,7(id 10),8,8(id 7),9
    assert r["order"].tolist() == [0, 1, 2, 3, 4, 8, 5, 10, 6, 7, 9]
    assert (r["d1"], r["A"]) == (1, 7 / 16)
    assert (r["d2"], r["B"]) == (5, 5 / 16)
    assert r["stop"] is False
    assert np.flatnonzero(r["active"]).tolist() == [1, 3, 5, 7, 10]


def test_stop_on_equality_and_not_below():
    """R4 with A == B stops ("<=" as written); B just below A does not."""
    al = _alpha()
    # k=1, h=1: C = {0}, M = {1}, F = {2, 3}; all T = 32 (alpha 2/16)
    for v2, stop in ((7, True), (8, True), (6, False)):
        S, T = _state([(32, 3), (32, 4), (32, v2), (32, 9)])
        r = orc.round_step(S, T, D, 1, 1, al)
        assert r["A"] == 5 / 16 and r["B"] == (v2 - 2) / 16
        assert r["stop"] is stop
        if stop:  # a stopped query still reports its blocker set: empty by construction
            assert not r["active"].any()


def test_d1_d2_ties_go_to_the_smaller_id_not_the_rank():
    """Equal U in C (and equal L in F) resolve to the smaller id even when the larger
    id ranks first."""
    al = _alpha()
    arms = [
        (64, 4),  # 0 C rank 2 (v=4): U = 5
        (32, 3),  # 1 C rank 1 (v=3): U = 5  -> tie, smaller id 0 wins
        (64, 5),  # 2 M
        (32, 7),  # 3 F rank 5 (v=7): L = 5  -> tie, smaller id 3 wins
        (64, 6),  # 4 F rank 4 (v=6): L = 5
        (64, 12),  # 5 F
    ]
    S, T = _state(arms)
    r = orc.round_step(S, T, D, 2, 1, al)
    assert r["order"].tolist() == [1, 0, 2, 4, 3, 5]
    assert (r["d1"], r["A"]) == (0, 5 / 16)
    assert (r["d2"], r["B"]) == (3, 5 / 16)
    assert r["stop"] is True


def test_h0_has_no_middle_band():
    """h = 0 (LUCB): ranks k+1.. are all F."""
    S, T = _state([(32, 2), (32, 3), (16, 4), (64, 9)])
    r = orc.round_step(S, T, D, 2, 0, _alpha())
    # C = {0, 1}: A = max(4, 5) = 5 (d1 = 1); F = {2, 3}: L = 0, 8 -> B = 0 (d2 = 2)
    assert (r["d1"], r["d2"], r["A"], r["B"]) == (1, 2, 5 / 16, 0.0)
    # blockers: C U > 0 -> 0, 1; F L < 5 -> 2 (L=0), not 3 (L=8)
    assert np.flatnonzero(r["active"]).tolist() == [0, 1, 2]


# --------------------------------------------------------------------------- Algorithm 1
def _constant_rows(values, d):
    """Points whose d coordinates all equal one value: every sampled coordinate gives the
    same squared difference, so after any T draws S = T (c - q)^2 whatever the RNG drew --
    the A1 trajectory is then fixed by hand."""
    return np.repeat(np.asarray(values, np.uint8)[:, None], d, axis=1)


def _a1_alpha(d):
    """alpha(u) = 0.5 / sqrt(u): a hand-made radius table (an input, R3)."""
    al = np.zeros(d + 1)
    al[1:d] = 0.5 / np.sqrt(np.arange(1, d))
    return al


def test_a1_b2_tie_goes_to_d2_then_smaller_id():
    """Eq. (4), b2 = argmax_{{d2} u M} alpha; ties to d2, then the smaller id.

    q = 0 and constant rows: d_hat_i = c_i^2 / 65025 whatever the draws; alpha(u) = 0.5/sqrt(u).
    c = (0, 10, 21, 20, 30, 200, 250) for ids 0..6; k = 2, h = 2.  Rank order by d_hat:
    0, 1, 3 (c=20), 2 (c=21), 4, 5, 6: C = {0, 1}, M = {3, 2} (larger id first), F = {4, 5, 6}.
    Iteration 1 (all T = 1, every alpha = 0.5): d1 = 1 (largest U in C), d2 = 4 (smallest L
      in F); M ties d2's alpha -> b2 = d2 = 4.  Draws on arms 1 and 4.
    Iteration 2: U_0 = 0 + 0.5 > U_1 = 0.0015 + 0.3536 -> d1 = 0; L_4 = 0.0138 - 0.3536 <
      L_5 = 0.6151 - 0.5 < L_6 -> d2 = 4 with alpha(2) = 0.3536; M arms 3 and 2 both have
      alpha(1) = 0.5 > 0.3536 and tie with each other -> the smaller id, 2 (not 3, which
      ranks first in M).  Draws on arms 0 and 2."""
    d = 64
    X = _constant_rows([0, 10, 21, 20, 30, 200, 250], d)
    x = np.zeros(d, np.uint8)
    al = _a1_alpha(d)
    r1 = orc.query_a1(X, x, 2, 2, 0, al, max_iters=2)  # iteration 1 samples; 2 hits the cap
    assert r1["status"] == orc.EMAXROUNDS
    assert r1["counts"].tolist() == [1, 2, 1, 1, 2, 1, 1]
    r2 = orc.query_a1(X, x, 2, 2, 0, al, max_iters=3)
    assert r2["counts"].tolist() == [2, 2, 2, 1, 2, 1, 1]
    for r in (r1, r2):
        assert np.array_equal(r["sums"], r["counts"].astype(np.int64) * X[:, 0].astype(np.int64) ** 2)


def test_a1_h0_b2_is_d2():
    """h = 0: the middle band is empty and b2 = d2 always (S:163 example).

    c = (0, 10, 30, 200), k = 1: C = {0}, F = {1, 2, 3}.
    It. 1: d1 = 0, d2 = 1 (L = 0.0015 - 0.5)          -> T = (2, 2, 1, 1)
    It. 2: L_1 = 0.0015 - 0.3536, L_2 = 0.0138 - 0.5  -> d2 = 2 -> T = (3, 2, 2, 1)
    It. 3: L_1 = 0.0015 - 0.3536 = -0.3520 < L_2 = 0.0138 - 0.3536 = -0.3397 -> d2 = 1
                                                      -> T = (4, 3, 2, 1)"""
    d = 64
    X = _constant_rows([0, 10, 30, 200], d)
    x = np.zeros(d, np.uint8)
    al = _a1_alpha(d)
    want = {2: [2, 2, 1, 1], 3: [3, 2, 2, 1], 4: [4, 3, 2, 1]}
    for cap, counts in want.items():
        r = orc.query_a1(X, x, 1, 0, 0, al, max_iters=cap)
        assert r["status"] == orc.EMAXROUNDS
        assert r["counts"].tolist() == counts, cap


def test_a1_d1_and_b2_are_never_the_same_arm():
    """SPEC.md:268 ("when d1 = b2 the arm receives two samples") cannot occur: d1 ranges
    over ranks 1..k and b2 over {d2} u ranks k+1..k+h, with d2 in ranks k+h+1..n -- disjoint
    rank ranges (reading R11).  So every iteration that does not stop draws ONE
    sample on each of two DIFFERENT arms: with d = 48 and <= 12 iterations no arm can reach
    T = d, so draws = n + 2 (iterations - 1) and consecutive caps differ by +1 on two arms."""
    rng = np.random.default_rng(5)
    n, d = 40, 48
    for trial in range(6):
        X = rng.integers(0, 256, (n, d), dtype=np.uint8)
        x = rng.integers(0, 256, d, dtype=np.uint8)
        al = orc.alpha_experimental(n, 0.05, d, 0.5)
        prev = None
        for it in range(1, 13):
            r = orc.query_a1(X, x, 3, 2 * (trial % 2), trial, al, max_iters=it)
            if r["status"] != orc.EMAXROUNDS:
                break
            assert r["draws"] == n + 2 * (it - 1)
            if prev is not None:
                diff = r["counts"] - prev["counts"]
                assert diff.min() == 0 and diff.max() == 1 and diff.sum() == 2
            prev = r
        assert prev is not None and prev["draws"] > n
