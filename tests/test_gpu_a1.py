"""GPU parity of the literal Algorithm 1 schedule.

aknn_query_a1 (one warp per query, a1_kernels.cu) against the oracle's A1 mode
(oracle/aknn_oracle.c orc_query_a1, one full sort per iteration): sets in rank
order, per-arm counts T_i and sums S_i, draws, evals and the iteration count
bit-exact; d_hat of the set to 0 ulp (the oracle side recomputes it from its own
S and T with the pinned expression S / (T * 65025.0), reading R15)."""
import numpy as np
import pytest

import oracle.oracle as orc
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ak():
    import torch
    torch.cuda.set_device(0)
    import paper_1902_09465_b200 as m
    return m


def _oracle_a1(X, Q, k, h, seed, alpha, max_iters=0):
    rows = [orc.query_a1(X, Q[qi], k, h, seed, alpha, qi=qi, max_iters=max_iters)
            for qi in range(Q.shape[0])]
    sets = np.stack([r["set"] for r in rows])
    sums = np.stack([r["sums"] for r in rows])
    counts = np.stack([r["counts"] for r in rows])
    dh = np.take_along_axis(sums, sets, 1).astype(np.float64) / (
        np.take_along_axis(counts, sets, 1).astype(np.float64) * 65025.0)
    return dict(sets=sets, counts=counts, sums=sums, dhat=dh,
                evals=np.array([r["evals"] for r in rows], np.int64),
                draws=np.array([r["draws"] for r in rows], np.int64),
                rounds=np.array([r["iters"] for r in rows], np.int32),
                status=[r["status"] for r in rows])


def _check(got, ref):
    for key in ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds"):
        g, r = got[key], ref[key]
        assert g.shape == r.shape, (key, g.shape, r.shape)
        if not np.array_equal(g, r):
            bad = np.argwhere(np.atleast_1d(g != r))[:5]
            raise AssertionError(f"{key} differs at {bad.tolist()}")


def _run(ak, X, Q, k, h, seed, alpha, max_iters=0):
    ix = ak.Index(X)
    try:
        got = ix.query(Q, k, h, 0.05, seed, alpha, counts=True, sums=True, schedule="a1",
                       max_rounds=max_iters)
    finally:
        ix.close()
    return got, _oracle_a1(X, Q, k, h, seed, alpha, max_iters)


@pytest.mark.parametrize("kind", ["exp0.1", "theory"])
def test_a1_config1_planted(ak, kind):
    """Config 1 (tiny planted instance): bit-exact, and the set is the 10 planted points."""
    cfg = synth.config(1)
    X, Q, planted = synth.planted(cfg)
    al = (orc.alpha_theory(cfg.n, cfg.delta, cfg.d) if kind == "theory"
          else orc.alpha_experimental(cfg.n, cfg.delta, cfg.d, 0.1))
    got, ref = _run(ak, X, Q, cfg.k, cfg.h, cfg.seed, al)
    _check(got, ref)
    assert sorted(got["sets"][0].tolist()) == planted.tolist()


A1_CASES = [
    # (name, n, d, q, k, h, alpha kind, c_alpha, seed, data kind)
    ("ragged", 333, 40, 3, 3, 4, "exp", 0.05, 1, "mixture"),
    ("d_not32", 211, 17, 4, 2, 3, "theory", 0, 2, "mixture"),
    ("h0_lucb", 150, 24, 3, 4, 0, "exp", 0.1, 3, "mixture"),
    ("uniform", 257, 32, 2, 5, 5, "exp", 0.2, 4, "uniform"),
    ("tiny_n", 6, 8, 3, 2, 3, "theory", 0, 5, "uniform"),
    ("d1", 50, 1, 2, 3, 3, "theory", 0, 6, "uniform"),
    ("d2", 64, 2, 3, 3, 3, "exp", 0.1, 7, "uniform"),
    ("wide_band", 700, 12, 2, 60, 50, "exp", 0.1, 8, "mixture"),
    # 4000 arms x 25 B > A1_SMEM_MAX: the state lives in the global workspace
    ("global_state", 4000, 4, 2, 3, 3, "exp", 0.01, 9, "mixture"),
    # the state (600 x 25 B) fits a CTA but not with the alpha / query tables of
    # d = 9000: global workspace (a launch-mode regression)
    ("tables_global", 600, 9000, 2, 3, 3, "exp", 0.001, 10, "mixture"),
]


@pytest.mark.parametrize("case", A1_CASES, ids=[c[0] for c in A1_CASES])
def test_a1_small_instances_bit_exact(ak, case):
    name, n, d, q, k, h, kind, c, seed, data = case
    X, Q = synth.small_instance(300 + seed, n, d, q=q, kind=data)
    al = orc.alpha_theory(n, 0.05, d) if kind == "theory" else orc.alpha_experimental(n, 0.05, d, c)
    got, ref = _run(ak, X, Q, k, h, 0xA1A1000000000000 + seed, al)
    _check(got, ref)
    assert got["status"] == 0


def test_a1_iteration_cap(ak):
    """max_rounds caps the iterations: AKNN_EMAXROUNDS with the state the oracle reaches."""
    X, Q = synth.small_instance(350, 400, 64, q=3)
    al = orc.alpha_theory(400, 0.05, 64)
    got, ref = _run(ak, X, Q, 4, 4, 9, al, max_iters=57)
    _check(got, ref)
    assert got["status"] == ak.AKNN_EMAXROUNDS
    assert (got["rounds"] == 57).all()


def test_a1_rejects_wide_band(ak):
    X, Q = synth.small_instance(351, 800, 8, q=1)
    ix = ak.Index(X)
    try:
        with pytest.raises(ak.AknnError):
            ix.query(Q, 300, 213, 0.05, 0, orc.alpha_theory(800, 0.05, 8), schedule="a1")
    finally:
        ix.close()


def test_a1_device_api_matches_host(ak):
    """aknn_query_a1_device (device buffers, a stream) gives the host call's bytes."""
    import torch
    X, Q = synth.small_instance(352, 300, 48, q=5)
    al = orc.alpha_experimental(300, 0.05, 48, 0.05)
    ix = ak.Index(torch.from_numpy(X).cuda())
    try:
        host = ix.query(Q, 3, 3, 0.05, 11, al, counts=True, sums=True, schedule="a1", qi_offset=7)
        dev = ix.query_device(torch.from_numpy(Q).cuda(), 3, 3, 0.05, 11, torch.from_numpy(al).cuda(),
                              counts=True, sums=True, schedule="a1", qi_offset=7)
        st = ix.stats()
    finally:
        ix.close()
    for key in ("sets", "dhat", "counts", "sums", "evals", "draws", "rounds"):
        assert np.array_equal(dev[key].cpu().numpy(), host[key]), key
    assert st["kernel_launches"] == 1
