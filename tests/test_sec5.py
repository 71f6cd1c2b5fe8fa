"""The paper's §5 workloads.

CPU (not gpu): the generator follows P:349 (x = c Q y on a p-dimensional subspace,
c the largest scalar with ||x||_inf <= 1/2 over the set) and the oracle reproduces
Figure 2's qualitative claims: on p = 10 the adaptive algorithm returns all
k nearest neighbours with a small fraction of the naive algorithm's coordinate
evaluations, and the saving shrinks as p grows.

GPU: the batched rule and the literal Algorithm 1 on full-size §5 trials (n = 1,000,
m = 12,288, k = h = 10, delta = 0.001, §5 alpha) bit-exact against the oracle.
"""
import numpy as np
import pytest

import oracle.oracle as orc
import synth

P = synth.SEC5


def _recall(X, q, got, k):
    D = ((X.astype(np.int64) - q.astype(np.int64)) ** 2).sum(1)
    dk = np.sort(D)[k - 1]
    s = D[np.asarray(got)]
    below = int((s < dk).sum())
    return (below + min(int((s == dk).sum()), k - below)) / k


@pytest.fixture(scope="module")
def p10():
    return synth.sec5_trial("p10", 0)


def test_generator_scale_hits_the_bound(p10):
    # c is the LARGEST scalar with ||x||_inf <= 1/2: some coordinate of the
    # set sits at +-1/2, i.e. at byte 0 or 255 after u = rint(255 (x + 1/2)).
    X, q = p10
    full = np.vstack([X, q])
    assert full.min() == 0 or full.max() == 255
    assert X.shape == (P["n"], P["m"]) and q.shape == (1, P["m"])


@pytest.mark.parametrize("p", [10, 100])
def test_generator_is_low_dimensional(p):
    # x = c Q y with Q in R^{m x p}: the set spans a p-dimensional subspace (through the
    # origin, which maps to byte 127.5); quantisation adds ~1/12 per coordinate.
    X, q = synth.subspace_trial(p, 0, n=400, m=2048)
    Z = np.vstack([X, q]).astype(np.float64) - 127.5
    sv = np.linalg.svd(Z, compute_uv=False)
    energy = np.cumsum(sv ** 2) / np.sum(sv ** 2)
    assert energy[p - 1] > 0.99
    assert energy[p // 2 - 1] < 0.99  # and not lower-dimensional than p


def test_generator_deterministic_and_trials_independent():
    a = synth.subspace_trial(10, 3, n=50, m=256)
    b = synth.subspace_trial(10, 3, n=50, m=256)
    c = synth.subspace_trial(10, 4, n=50, m=256)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[0], c[0])
    X, q = synth.images_trial(1, n=30)
    assert X.shape == (30, 12_288) and X.dtype == np.uint8


def test_figure2_claims_on_the_oracle():
    """p = 10 -> all k-NN returned at a small fraction; p = 1000 -> little
    saving at the same C_alpha (batched rule, which samples at least as much as
    Algorithm 1's schedule)."""
    c = 1e-4
    out = {}
    for w in ("p10", "p1000"):
        X, q = synth.sec5_trial(w, 0)
        al = orc.alpha_experimental(P["n"], P["delta"], P["m"], c)
        r = orc.query_br(X, q, P["k"], P["h"], 0, al)
        out[w] = (_recall(X, q[0], r["sets"][0], P["k"]), r["evals"][0] / (P["n"] * P["m"]))
    assert out["p10"][0] == 1.0
    assert out["p10"][1] < 0.25
    assert out["p1000"][1] > 5 * out["p10"][1]


def test_a1_samples_less_than_br_on_p10(p10):
    X, q = p10
    al = orc.alpha_experimental(P["n"], P["delta"], P["m"], 1e-5)
    a = orc.query_a1(X, q[0], P["k"], P["h"], 0, al)
    b = orc.query_br(X, q, P["k"], P["h"], 0, al)
    assert a["status"] == 0
    assert a["evals"] < b["evals"][0] / 2


# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def ak():
    import torch
    torch.cuda.set_device(0)
    import paper_1902_09465_b200 as m
    return m


@pytest.mark.gpu
@pytest.mark.parametrize("w,trial,c,sched", [
    ("p10", 0, 1e-5, "a1"), ("p10", 0, 1e-4, "br"), ("p1000", 1, 1e-4, "br"),
    ("images", 0, 1e-3, "a1"), ("images", 2, 1e-3, "br"), ("p10", 3, 1e-3, "br_g2"),
    ("p100", 4, 1e-4, "br_g2")])
def test_gpu_sec5_bit_exact(ak, w, trial, c, sched):
    X, q = synth.sec5_trial(w, trial)
    n, m, k, h = P["n"], P["m"], P["k"], P["h"]
    al = orc.alpha_experimental(n, P["delta"], m, c)
    ix = ak.Index(X)
    try:
        g2 = sched == "br_g2"  # growth factor < 2 (reading R25)
        got = ix.query(q, k, h, P["delta"], trial, al, counts=True, sums=True,
                       schedule="br" if g2 else sched, growth=2 if g2 else 1)
    finally:
        ix.close()
    if sched == "a1":
        r = orc.query_a1(X, q[0], k, h, trial, al)
        assert got["status"] == r["status"] == 0
        assert np.array_equal(got["sets"][0], r["set"])
        assert np.array_equal(got["counts"][0], r["counts"])
        assert np.array_equal(got["sums"][0], r["sums"])
        assert (got["evals"][0], got["draws"][0], got["rounds"][0]) == (r["evals"], r["draws"], r["iters"])
    else:
        r = orc.query_br(X, q, k, h, trial, al, want_sums=True, growth=2 if g2 else 1)
        for key in ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds"):
            assert np.array_equal(got[key], r[key]), key
