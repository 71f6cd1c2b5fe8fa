"""Pins of the oracle's close-side lead (reading R24):
with lead L > 1, the blockers of a round that rank in C or M advance L times (each the
P:176 / doubling step), the far blockers once.

Pinned by what the schedule cannot change: every arm still sums the first T of its own
(cuRAND-pinned) sample stream, exact arms hold the brute-force distance, the returned
set contains the exact k nearest neighbours (P:395-399 holds under any schedule), and
L = 1 is the batched rule itself."""
import numpy as np
import pytest

import oracle.oracle as orc
import synth


def test_lead_one_is_the_batched_rule():
    X, Q = synth.small_instance(701, 400, 64, q=3)
    al = orc.alpha_experimental(400, 0.05, 64, 0.1)
    a = orc.query_br(X, Q, 4, 4, 2, al, want_sums=True)
    b = orc.query_br(X, Q, 4, 4, 2, al, want_sums=True, lead=1)
    for key in ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("lead", [2, 3, 5])
def test_lead_sums_are_the_arm_streams(lead):
    X, Q = synth.small_instance(702, 150, 40, q=2)
    n, d = X.shape
    seed = 9
    al = orc.alpha_experimental(n, 0.05, d, 0.05)
    r = orc.query_br(X, Q, 3, 3, seed, al, want_sums=True, lead=lead)
    D = ((X[None].astype(np.int64) - Q[:, None].astype(np.int64)) ** 2).sum(2)
    for a in range(2):
        for i in range(n):
            T = int(r["counts"][a, i])
            if T == d:
                assert r["sums"][a, i] == D[a, i]
            else:
                js = [orc.draw_index(seed, a, i, t, d) for t in range(T)]
                want = int(((X[i, js].astype(np.int64) - Q[a, js].astype(np.int64)) ** 2).sum())
                assert r["sums"][a, i] == want


@pytest.mark.parametrize("lead", [2, 4])
def test_lead_keeps_the_knn_guarantee(lead):
    fails = 0
    for s in range(30):
        X, Q = synth.small_instance(710 + s, 200, 48, q=2)
        al = orc.alpha_theory(200, 0.05, 48)
        r = orc.query_br(X, Q, 5, 5, s, al, lead=lead)
        idx, _ = orc.bruteforce(X, Q, 5)
        for a in range(2):
            fails += not set(idx[a].tolist()) <= set(r["sets"][a].tolist())
    assert fails <= 3  # delta = 0.05 over 60 queries (Theorem 1); in practice 0


def test_lead_moves_close_arms_further_per_round():
    """The C/M blockers are the arms near the boundary: with a lead they reach the
    levels that decide Eq. (5) in fewer rounds, and the far arms double fewer times
    (C1, C_alpha = 0.1)."""
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_experimental(cfg.n, cfg.delta, cfg.d, 0.1)
    base = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al)
    led = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, lead=3)
    assert sorted(led["sets"][0].tolist()) == planted.tolist()
    assert led["rounds"][0] <= base["rounds"][0]
    assert led["evals"][0] < base["evals"][0]
