"""GPU parity (-m gpu) of the exact comparison pass (row a10): aknn_exact against
the oracle's brute force (orc_bruteforce: all exact distances, sorted by (distance,
smaller id)) -- indices and squared distances element by element.

k <= 128 runs the fused tcgen05 kernel with the running top-k epilogue
(exact_fused.cu); k > 128 the distance-matrix path (exact_mma.cu + block top-k).
Cases: ragged q / n / d around the 128 x 256 tiles and 128-byte k-blocks, ties, k = 1,
k = 128, k = n, many point ranges per query block, more query blocks than SMs (several
launches), a sharded index (global ids), and the BASELINE sizes of configs 2 and 4 on
sampled queries."""
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


def _check(ak, X, Q, k, rows=None, offset=0, n_global=None):
    ix = ak.Index(X) if n_global is None else ak.Index(X, n_global=n_global, offset=offset)
    idx, dist = ix.exact(Q, k)
    ix.close()
    Qr = Q if rows is None else Q[rows]
    ridx, rdist = orc.bruteforce(X, Qr, k)
    gi, gd = (idx, dist) if rows is None else (idx[rows], dist[rows])
    assert np.array_equal(gd, rdist), np.argwhere(gd != rdist)[:5].tolist()
    assert np.array_equal(gi, ridx + offset), np.argwhere(gi != ridx + offset)[:5].tolist()


CASES = [
    # name, n, d, q, k, value range (small ranges force distance ties)
    ("tiny_one_tile", 200, 64, 3, 5, 256),
    ("k_equals_n", 40, 17, 5, 40, 256),
    ("k1", 3000, 300, 7, 1, 256),
    ("k128_ragged", 5003, 129, 130, 128, 256),
    ("ties_binary", 9000, 48, 33, 50, 2),
    ("ties_ternary_k100", 20011, 255, 260, 100, 3),
    ("d_one_byte_per_block", 4097, 1, 5, 7, 256),
    ("d_768_many_ranges", 70000, 768, 300, 100, 256),
    ("d_12288_wide_rows", 3000, 12288, 129, 10, 256),
    ("k_above_fused_cap", 6000, 96, 70, 200, 256),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_exact_vs_bruteforce(ak, case):
    _, n, d, q, k, hi = case
    rng = np.random.default_rng(n * 7 + d)
    X = rng.integers(0, hi, (n, d), dtype=np.uint8)
    Q = rng.integers(0, hi, (q, d), dtype=np.uint8)
    _check(ak, X, Q, k)


def test_more_query_blocks_than_sms(ak):
    """q > 148 * 128: the fused pass runs in several launches (chunks of m-blocks)."""
    rng = np.random.default_rng(11)
    n, d, q, k = 700, 40, 148 * 128 + 300, 9
    X = rng.integers(0, 256, (n, d), dtype=np.uint8)
    Q = rng.integers(0, 256, (q, d), dtype=np.uint8)
    rows = np.concatenate([np.arange(0, 5), rng.choice(q, 40, replace=False), np.arange(q - 5, q)])
    _check(ak, X, Q, k, rows=rows)


def test_sharded_index_reports_global_ids(ak):
    rng = np.random.default_rng(12)
    X = rng.integers(0, 256, (3000, 64), dtype=np.uint8)
    Q = rng.integers(0, 256, (9, 64), dtype=np.uint8)
    _check(ak, X, Q, 12, offset=5000, n_global=10000)


def test_config2_full_size(ak):
    """Config 2 at its BASELINE size (n = 60,000, d = 784, all 1,000 queries in one call);
    64 sampled queries recomputed by the oracle's brute force."""
    cfg = synth.config(2)
    X, Q = synth.points(cfg), synth.queries(cfg)
    rows = np.random.default_rng(2).choice(cfg.q, 64, replace=False)
    _check(ak, X, Q, cfg.k, rows=rows)


def test_config4_full_size(ak):
    """Config 4 at its BASELINE size (n = 1,000,000, d = 1,024, 128 queries, k = 50);
    3 sampled queries recomputed by the oracle's brute force."""
    cfg = synth.config(4)
    X, Q = synth.points(cfg), synth.queries(cfg)
    rows = np.random.default_rng(4).choice(cfg.q, 3, replace=False)
    _check(ak, X, Q, cfg.k, rows=rows)


def test_distance_matrix_path_multi_chunk(ak):
    """k > 128 with q * npad * 4 B > 2 GiB: the distance-matrix path in several query
    chunks; sampled queries from both chunks."""
    rng = np.random.default_rng(13)
    n, d, q, k = 1_100_000, 16, 520, 129
    X = rng.integers(0, 256, (n, d), dtype=np.uint8)
    Q = rng.integers(0, 256, (q, d), dtype=np.uint8)
    _check(ak, X, Q, k, rows=np.array([0, 1, 487, 488, 519]))
