"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a library routine, a closed
form, a worked example in SPEC.md/PAPER.md (tests/golden/), an invariant, or
brute force on tiny inputs.  See DESIGN.md §4 for the pin table.
"""
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

import oracle.oracle as orc
import synth

HERE = os.path.dirname(os.path.abspath(__file__))


# --------------------------------------------------------------------------- a1: RNG
def _curand_philox(lines):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available to build the cuRAND pin helper")
    tmp = tempfile.mkdtemp()
    exe = os.path.join(tmp, "curand_philox")
    subprocess.check_call([nvcc, "-Wno-deprecated-gpu-targets", "-o", exe,
                           os.path.join(HERE, "cpin", "curand_philox.cu")])
    out = subprocess.run([exe], input="\n".join(" ".join(map(str, l)) for l in lines),
                         capture_output=True, text=True, check=True).stdout
    return [list(map(int, l.split())) for l in out.strip().splitlines()]


def test_philox_matches_curand_library_routine():
    """Philox4x32-10 == cuRAND curand_Philox4x32_10 (library routine, host-evaluated)."""
    rng = np.random.default_rng(123)
    lines = [[0, 0, 0, 0, 0, 0], [1, 2, 3, 4, 5, 6],
             [0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF]]
    lines += rng.integers(0, 2**32, (200, 6), dtype=np.uint64).tolist()
    ref = _curand_philox(lines)
    for l, r in zip(lines, ref):
        got = orc.philox4x32_10(l[:4], l[4:]).tolist()
        assert got == r, (l, got, r)


@pytest.mark.parametrize("d", [784, 12288])
def test_lemire_exhaustive_preimage_counts(d):
    """Every j in [0,d) has floor(2^32/d) or ceil(2^32/d) preimages (closed form),
    and the counts sum to 2^32 (brute force over all words)."""
    h = orc.lemire_histogram(d)
    lo, hi = (2**32) // d, -(-(2**32) // d)
    assert int(h.sum()) == 2**32
    assert int(h.min()) >= lo and int(h.max()) <= hi
    # number of j receiving the larger count is fixed: 2^32 mod d
    assert int((h == hi).sum()) == (2**32) % d or lo == hi


def test_lemire_power_of_two_is_top_bits():
    """For d = 2^b the multiply-high map is the top b bits of the word (closed form)."""
    rng = np.random.default_rng(1)
    for b in (1, 8, 10):
        for w in rng.integers(0, 2**32, 50).tolist():
            assert orc.lemire(w, 2**b) == w >> (32 - b)


def test_draw_counter_layout_levels():
    """Draw(i,t) uses counter (u>>2, i, qi, b) with b = 0 for t=0 else 1+floor(log2 t),
    u = t - 2^(b-1); checked against Philox + Lemire evaluated here."""
    seed = 0x1234_5678_9ABC_DEF0
    key = [seed & 0xFFFFFFFF, seed >> 32]
    d = 784
    for qi, i in [(0, 0), (3, 17), (999, 59999)]:
        for t in [0, 1, 2, 3, 4, 5, 7, 8, 15, 16, 100, 511, 4096]:
            b = 0 if t == 0 else 1 + int(math.floor(math.log2(t)))
            u = t - (0 if b == 0 else 2 ** (b - 1))
            w = orc.philox4x32_10([u >> 2, i, qi, b], key)[u & 3]
            assert orc.draw_index(seed, qi, i, t, d) == (int(w) * d) >> 32


def test_draws_uniform_chi_square():
    """Sampled coordinates are uniform on [m]: chi-square over 20000 draws, m=10."""
    d = 10
    js = np.array([orc.draw_index(7, 1, 2, t, d) for t in range(20000)])
    cnt = np.bincount(js, minlength=d)
    chi2 = float(((cnt - 2000.0) ** 2 / 2000.0).sum())
    assert chi2 < 40.0  # 9 dof; p ~ 5e-6


def test_single_sample_unbiased():
    """E[(x_j - q_j)^2] = D_i (P:393 'E[d_hat_i(t)] = d_i'): Monte-Carlo mean of 40000
    draws within 5 sigma of the exact mean (brute force)."""
    rng = np.random.default_rng(5)
    d = 97
    x = rng.integers(0, 256, d)
    y = rng.integers(0, 256, d)
    sq = (x - y) ** 2
    js = np.array([orc.draw_index(11, 0, 3, t, d) for t in range(40000)])
    mean = sq[js].mean()
    sd = sq.std() / math.sqrt(len(js))
    assert abs(mean - sq.mean()) < 5 * sd


# --------------------------------------------------------------------------- alpha
def _golden_alpha():
    rows = []
    with open(os.path.join(HERE, "golden", "alpha_worked.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            p = line.split()
            rows.append(dict(variant=p[0], n=int(p[1]), delta=float(p[2]), c=float(p[3]),
                             u=int(p[4]), value=float(p[5]), tol=float(p[6])))
    return rows


@pytest.mark.parametrize("row", _golden_alpha(),
                         ids=lambda r: f"{r['variant']}-n{r['n']}-u{r['u']}-c{r['c']}")
def test_alpha_worked_values(row):
    """Worked values of alpha(u): SPEC.md:78-79 at u = 1, hand derivations at u > 1
    (the u-dependent term 1.5 log(1 + log u) of footnote 2 and (1 + log u) of §5), and
    the survey-time values at each config's last sampled level."""
    d = max(16, row["u"] + 1)
    if row["variant"] == "theory":
        a = orc.alpha_theory(row["n"], row["delta"], d)
    else:
        a = orc.alpha_experimental(row["n"], row["delta"], d, row["c"])
    assert abs(a[row["u"]] - row["value"]) <= row["tol"]


@pytest.mark.parametrize("n,d,delta", [(1000, 256, 0.05), (60000, 784, 0.05),
                                       (100000, 12288, 0.05), (8_000_000, 768, 0.01)])
def test_alpha_table_shape_and_monotone(n, d, delta):
    """alpha is strictly decreasing on [1, d), alpha(4u) < alpha(u),
    alpha(u)*sqrt(u) grows only logarithmically, and alpha[d] = 0."""
    for a in (orc.alpha_theory(n, delta, d), orc.alpha_experimental(n, delta, d, 1.0)):
        assert a[d] == 0.0
        assert np.all(np.diff(a[1:d]) < 0)
        r = a[1:d] * np.sqrt(np.arange(1, d))
        assert np.all(np.diff(r) >= 0) and r[-1] / r[0] < 1.5


def test_alpha_theory_undefined_region():
    """delta/n >= 1/e leaves log log(1/delta') undefined or <= 0: rejected."""
    with pytest.raises(ValueError):
        orc.alpha_theory(1, 0.5, 8)


def test_alpha_lemma1_coverage_monte_carlo():
    """Lemma 1: with Theory alpha, |d_hat(t) - D| <= alpha(t) for all t < m,
    for every arm, in >= 1 - delta of runs.  Simulated on Bernoulli-like bounded samples."""
    rng = np.random.default_rng(2)
    n, m, delta = 20, 512, 0.1
    a = orc.alpha_theory(n, delta, m)
    fails = 0
    runs = 200
    for _ in range(runs):
        p = rng.uniform(0, 1, n)
        s = (rng.uniform(0, 1, (n, m - 1)) < p[:, None]).astype(float)
        est = np.cumsum(s, axis=1) / np.arange(1, m)
        if np.any(np.abs(est - p[:, None]) > a[1:m][None, :]):
            fails += 1
    assert fails / runs <= delta


# --------------------------------------------------------------------------- brute force
def test_bruteforce_matches_numpy_and_int_mm():
    """orc_bruteforce == numpy int64 sums (stable sort by (D, i)) == torch._int_mm form."""
    import torch
    X, Q = synth.small_instance(3, 500, 64, q=4)
    k = 12
    idx, dist = orc.bruteforce(X, Q, k)
    D = ((X[None].astype(np.int64) - Q[:, None].astype(np.int64)) ** 2).sum(-1)
    for a in range(Q.shape[0]):
        o = np.lexsort((np.arange(X.shape[0]), D[a]))[:k]
        assert idx[a].tolist() == o.tolist()
        assert dist[a].tolist() == D[a][o].tolist()
    xs = torch.from_numpy(X.astype(np.int16) - 128).to(torch.int8)
    qs = torch.from_numpy(Q.astype(np.int16) - 128).to(torch.int8)
    dot = torch._int_mm(torch.nn.functional.pad(qs, (0, 0, 0, 16 - 4)), xs.t().contiguous())[:4]
    nx = (xs.int() ** 2).sum(1)
    nq = (qs.int() ** 2).sum(1)
    D2 = (nq[:, None] + nx[None, :] - 2 * dot).numpy()
    assert np.array_equal(D2, D)


# --------------------------------------------------------------------------- round step
def _state(values_T, d=64):
    """Build S from exact decimal estimates: S = v * 65025 * T (integers by construction)."""
    S, T = [], []
    for v, t in values_T:
        s = v * 65025 * t
        assert abs(s - round(s)) < 1e-6
        S.append(int(round(s)))
        T.append(t)
    return np.array(S), np.array(T)


def test_partition_examples_spec():
    """n=4,k=1,h=1; sorted or all-equal estimates -> close={0}, mid={1}."""
    al = np.zeros(65)
    al[1:64] = 0.01
    for vals in ([0.1, 0.2, 0.3, 0.4], [0.5, 0.5, 0.5, 0.5]):
        S, T = _state([(v, 2) for v in vals])
        r = orc.round_step(S, T, 64, 1, 1, al)
        assert r["order"][0] == 0 and r["order"][1] == 1
        assert sorted(r["order"][2:].tolist()) == [2, 3]


def test_peek_d1_d2_examples_spec():
    """SPEC.md:149 (d1 = A since 0.6 > 0.25) and SPEC.md:159 (d2 = C since 0.1 < 0.4)."""
    al = np.zeros(65)
    al[2], al[4], al[8] = 0.5, 0.05, 0.1
    # close = {A(0): 0.1 @T=2 (a=.5), B(1): 0.2 @T=4 (a=.05)}; far = two arms at 0.9
    S, T = _state([(0.1, 2), (0.2, 4), (0.9, 8), (0.9, 8)])
    r = orc.round_step(S, T, 64, 2, 0, al)
    assert r["d1"] == 0 and abs(r["A"] - 0.6) < 1e-12
    # close = {0.05 @T=4}; far = {C(1): 0.9 @T=2 (a=.8), D(2): 0.5 @T=8 (a=.1)}
    al2 = np.zeros(65)
    al2[2], al2[4], al2[8] = 0.8, 0.05, 0.1
    S, T = _state([(0.05, 4), (0.9, 2), (0.5, 8)])
    r = orc.round_step(S, T, 64, 1, 0, al2)
    assert r["d2"] == 1 and abs(r["B"] - 0.1) < 1e-12


def test_all_far_exact_d2_is_smallest_far_distance():
    """all far arms exact (alpha=0) -> d2 = smallest exact distance in far."""
    d = 64
    al = np.full(d + 1, 0.3)
    al[d] = 0.0
    S = np.array([10, 5000, 4000, 9000, 4500]) * 1
    T = np.array([1, d, d, d, d])
    r = orc.round_step(S, T, d, 1, 0, al)
    assert r["d2"] == 2


def test_round_step_order_matches_brute_sort():
    """The permutation (.) equals a brute-force lexicographic sort of exact rationals
    S/(65025 T) with ties to the smaller index (Fraction arithmetic, not fp64)."""
    from fractions import Fraction
    rng = np.random.default_rng(9)
    d = 784
    T = rng.choice([1, 2, 4, 8, 16, d], 300)
    S = np.array([rng.integers(0, 65025 * t + 1) for t in T])
    S[:40] = S[40:80] * 1
    T[:40] = T[40:80]
    r = orc.round_step(S, T, d, 5, 5, orc.alpha_theory(300, 0.05, d))
    key = [(Fraction(int(s), 65025 * int(t)), i) for i, (s, t) in enumerate(zip(S, T))]
    assert r["order"].tolist() == [i for _, i in sorted(key)]


# --------------------------------------------------------------------------- BR
def _recall_ok(X, x, sets, k):
    """Tie rule (R16): all i with D_i < D_(k), plus enough of those tied at D_(k)."""
    D = ((X.astype(np.int64) - x.astype(np.int64)) ** 2).sum(1)
    Dk = np.sort(D)[k - 1]
    strict = set(np.nonzero(D < Dk)[0].tolist())
    tied = set(np.nonzero(D == Dk)[0].tolist())
    s = set(sets.tolist())
    return strict <= s and len(s & tied) >= k - len(strict)


def test_br_planted_config1_returns_planted_set():
    """Config 1: the 10 planted rows (D ~ 4e-4) vs the 11th nearest (~0.13): the
    returned k+h=10 set must equal the planted set, by construction."""
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    r = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al)
    assert sorted(r["sets"][0].tolist()) == planted.tolist()


def test_br_d_equals_1_is_exact_after_init():
    """m=1: the first sample is exact; Eq. (5) holds in round 1 and the set
    is the brute-force top-(k+h) in order, with d_hat = D/65025 to 0 ulp."""
    rng = np.random.default_rng(4)
    X = rng.integers(0, 256, (200, 1), dtype=np.uint8)
    Q = rng.integers(0, 256, (3, 1), dtype=np.uint8)
    k, h = 4, 3
    al = orc.alpha_theory(200, 0.05, 1)
    r = orc.query_br(X, Q, k, h, 0, al, want_sums=True)
    idx, dist = orc.bruteforce(X, Q, k + h)
    assert np.all(r["rounds"] == 1) and np.all(r["counts"] == 1)
    assert np.array_equal(r["sets"], idx)
    assert np.array_equal(r["dhat"], dist / 65025.0)
    assert np.all(r["evals"] == 200) and np.all(r["draws"] == 200)


def test_br_exact_arms_equal_brute_force():
    """Once T_i = m the estimate is the exact distance: S_i == brute-force D_i
    and d_hat == D/(m*65025) to 0 ulp for every exact arm."""
    X, Q = synth.small_instance(21, 300, 48, q=3)
    al = orc.alpha_theory(300, 0.05, 48)
    r = orc.query_br(X, Q, 5, 5, 3, al, want_sums=True)
    D = ((X[None].astype(np.int64) - Q[:, None].astype(np.int64)) ** 2).sum(-1)
    ex = r["counts"] == 48
    assert ex.sum() > 0
    assert np.array_equal(r["sums"][ex], D[ex])
    for a in range(3):
        for rank, i in enumerate(r["sets"][a]):
            if r["counts"][a, i] == 48:
                assert r["dhat"][a, rank] == D[a, i] / (48 * 65025.0)


def test_br_accounting_closed_forms():
    """T_i in {2^b : 2^b < m} u {m}; draws = sum_{T<m} T_i + #exact * T_prev with
    T_prev the smallest power of two with 2T >= m; evals = draws + m*#exact;
    rounds <= 1 + n*ceil(log2 m)  (SURVEY §8(c) guarantees)."""
    for seed, (n, d) in enumerate([(300, 48), (257, 100), (120, 33)]):
        X, Q = synth.small_instance(100 + seed, n, d, q=2)
        for al in (orc.alpha_theory(n, 0.05, d), orc.alpha_experimental(n, 0.05, d, 0.01)):
            r = orc.query_br(X, Q, 3, 4, seed, al)
            tprev = 1
            while 2 * tprev < d:
                tprev *= 2
            for a in range(2):
                T = r["counts"][a]
                samp = T[T < d]
                assert np.all((samp & (samp - 1)) == 0) and np.all(samp < d)
                nex = int((T == d).sum())
                assert r["draws"][a] == int(samp.sum()) + nex * tprev
                assert r["evals"][a] == r["draws"][a] + d * nex
                assert r["rounds"][a] <= 1 + n * math.ceil(math.log2(d))


def test_br_theorem1_failure_rate():
    """Theorem 1: under Theory alpha the returned set contains the k nearest
    neighbours in >= 1-delta of runs; 150 seeded instances, delta = 0.1."""
    delta = 0.1
    fails = 0
    runs = 150
    for s in range(runs):
        X, Q = synth.small_instance(1000 + s, 80, 24, q=1, centres=3, sigma=40.0)
        al = orc.alpha_theory(80, delta, 24)
        r = orc.query_br(X, Q, 3, 3, s, al)
        fails += not _recall_ok(X, Q[0], r["sets"][0], 3)
    assert fails / runs <= delta


def test_br_stops_with_eq5_and_sets_are_ranked():
    """At return, Eq. (5) holds on the final state and the set is (1)..(k+h) of (d_hat, i)."""
    X, Q = synth.small_instance(7, 400, 64, q=2)
    al = orc.alpha_experimental(400, 0.05, 64, 0.05)
    r = orc.query_br(X, Q, 6, 4, 9, al, want_sums=True)
    for a in range(2):
        st = orc.round_step(r["sums"][a], r["counts"][a], 64, 6, 4, al, want_active=False)
        assert st["stop"]
        assert st["order"][:10].tolist() == r["sets"][a].tolist()


def test_br_h0_is_lucb_bottom_k():
    """h = 0 degenerates to LUCB bottom-k: the set has k elements containing the
    exact k nearest neighbours (Theory alpha)."""
    X, Q = synth.small_instance(8, 150, 32, q=3)
    r = orc.query_br(X, Q, 4, 0, 1, orc.alpha_theory(150, 0.05, 32))
    for a in range(3):
        assert _recall_ok(X, Q[a], r["sets"][a], 4)


def test_br_query_order_and_determinism():
    """Identical inputs -> identical outputs; a query's result depends only on (X, x, qi)."""
    X, Q = synth.small_instance(12, 200, 40, q=3)
    al = orc.alpha_experimental(200, 0.05, 40, 0.1)
    r1 = orc.query_br(X, Q, 3, 3, 5, al, want_sums=True)
    r2 = orc.query_br(X, Q, 3, 3, 5, al, want_sums=True)
    for key in ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds"):
        assert np.array_equal(r1[key], r2[key])
    r3 = orc.query_br(X, Q[2:3], 3, 3, 5, al, qids=[2], want_sums=True)
    assert np.array_equal(r3["sums"][0], r1["sums"][2])


def _stream_sum(X, x, seed, qi, i, T):
    d = X.shape[1]
    js = [orc.draw_index(seed, qi, i, t, d) for t in range(T)]
    return int(((X[i, js].astype(np.int64) - x[js].astype(np.int64)) ** 2).sum())


def test_a1_and_br_share_per_arm_streams():
    """A1 (literal Algorithm 1) and BR both accumulate the same per-arm stream:
    for every sampled arm, S_i = sum_{t<T_i} (X[i][j_t] - x[j_t])^2 with j_t the pinned
    Draw(i, t) -- recomputed here from draw_index and numpy integer arithmetic."""
    X, Q = synth.small_instance(13, 40, 64, q=1)
    al = orc.alpha_experimental(40, 0.05, 64, 0.02)
    br = orc.query_br(X, Q, 2, 2, 77, al, want_sums=True)
    a1 = orc.query_a1(X, Q[0], 2, 2, 77, al)
    for counts, sums in ((br["counts"][0], br["sums"][0]), (a1["counts"], a1["sums"])):
        for i in range(40):
            if counts[i] < 64:
                assert sums[i] == _stream_sum(X, Q[0], 77, 0, i, int(counts[i]))
    same = (br["counts"][0] == a1["counts"]) & (a1["counts"] < 64)
    assert np.array_equal(br["sums"][0][same], a1["sums"][same])


def test_a1_literal_contains_knn():
    """A1 on tiny instances returns a set containing the k nearest neighbours (Theory alpha)."""
    for s in range(5):
        X, Q = synth.small_instance(200 + s, 30, 16, q=1)
        r = orc.query_a1(X, Q[0], 2, 2, s, orc.alpha_theory(30, 0.05, 16))
        assert _recall_ok(X, Q[0], r["set"], 2)


# ----------------------------------------------------------------- query-independent draws
# every query's Philox counter word is SHARED_QI, so arm i's t-th
# coordinate is the same for all queries.  Each query alone is still the paper's
# algorithm with i.i.d. uniform coordinates, so the same pins hold.

def test_shared_draws_planted_config1_returns_planted_set():
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    r = orc.query_br(X, Q, cfg.k, cfg.h, cfg.seed, al, shared_draws=True)
    assert sorted(r["sets"][0].tolist()) == planted.tolist()


def test_shared_draws_same_coordinates_for_every_query():
    """With shared draws two queries that agree on every coordinate but one, c, have
    per-arm sums that differ only through the draws landing on c: S1_i - S2_i ==
    n_c(i) * ((x_ic - q1_c)^2 - (x_ic - q2_c)^2) where n_c(i) = how many of arm i's T_i
    draws hit c -- so n_c(i) is the same for both queries (checked against the draw
    index, which is pinned to cuRAND's Philox above)."""
    X, Q = synth.small_instance(31, 200, 16, q=1)
    q1 = Q[0].copy()
    q2 = q1.copy()
    q2[5] = (int(q2[5]) + 97) % 256
    al = orc.alpha_experimental(200, 0.05, 16, 1e-6)  # tiny radius: stops early, T small
    r = orc.query_br(X, np.stack([q1, q2]), 3, 3, 9, al, want_sums=True, shared_draws=True,
                     max_rounds=1)
    T = r["counts"]
    assert np.array_equal(T[0], T[1])  # round 1: every arm has T = 1
    for i in range(200):
        t0 = 0
        hits = sum(orc.draw_index(9, orc.SHARED_QI, i, t, 16) == 5 for t in range(t0, T[0, i]))
        a = int(X[i, 5])
        want = hits * ((a - int(q1[5])) ** 2 - (a - int(q2[5])) ** 2)
        assert r["sums"][0, i] - r["sums"][1, i] == want


def test_shared_draws_identical_queries_identical_results():
    X, Q = synth.small_instance(33, 500, 40, q=1)
    al = orc.alpha_theory(500, 0.05, 40)
    QQ = np.repeat(Q, 3, axis=0)
    r = orc.query_br(X, QQ, 4, 4, 2, al, want_sums=True, shared_draws=True)
    for k in ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds"):
        assert np.array_equal(r[k][0], r[k][1]) and np.array_equal(r[k][0], r[k][2]), k
    d = orc.query_br(X, QQ, 4, 4, 2, al, want_sums=True)  # per-query streams differ
    assert not np.array_equal(d["sums"][0], d["sums"][1])


def test_shared_draws_exact_arms_and_theorem1():
    """Exact arms equal brute force; the Theorem-1 failure rate stays <= delta."""
    X, Q = synth.small_instance(21, 300, 48, q=3)
    al = orc.alpha_theory(300, 0.05, 48)
    r = orc.query_br(X, Q, 5, 5, 3, al, want_sums=True, shared_draws=True)
    D = ((X[None].astype(np.int64) - Q[:, None].astype(np.int64)) ** 2).sum(-1)
    ex = r["counts"] == 48
    assert ex.sum() > 0 and np.array_equal(r["sums"][ex], D[ex])
    delta, fails, runs = 0.1, 0, 100
    for s in range(runs):
        X, Q = synth.small_instance(2000 + s, 80, 24, q=1, centres=3, sigma=40.0)
        r = orc.query_br(X, Q, 3, 3, s, orc.alpha_theory(80, delta, 24), shared_draws=True)
        fails += not _recall_ok(X, Q[0], r["sets"][0], 3)
    assert fails / runs <= delta
