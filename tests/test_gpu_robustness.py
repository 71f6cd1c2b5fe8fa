"""GPU tests (-m gpu) of the round-1 advisor findings: sub-batching (qb < q) with and
without a round cap, sharded statistics, argument validation of the device and
multi-shard bindings, and the row-norm ordering across streams."""
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
        assert np.array_equal(got[k], ref[k]), k


@pytest.mark.parametrize("bq", [1, 3, 4])
def test_sub_batches_equal_one_batch_and_oracle(ak, bq):
    """batch_queries forces qb < q: several internal sub-batches (and graph shapes)."""
    X, Q = synth.small_instance(71, 2500, 120, q=10)
    al = orc.alpha_theory(2500, 0.05, 120)
    ix = ak.Index(X)
    one = ix.query(Q, 4, 5, 0.05, 21, al, sums=True)
    split = ix.query(Q, 4, 5, 0.05, 21, al, sums=True, batch_queries=bq)
    st = ix.stats()
    ix.close()
    assert st["query_batches"] == -(-10 // bq)
    _eq(split, one)
    ref = orc.query_br(X, Q, 4, 5, 21, al, want_sums=True)
    _eq(split, ref)


@pytest.mark.parametrize("timing", [False, True])
def test_sub_batches_with_round_cap_fill_every_row(ak, timing):
    """EMAXROUNDS in the first sub-batch no longer skips the later ones (stale rows)."""
    X, Q = synth.small_instance(72, 2000, 200, q=7)
    al = orc.alpha_theory(2000, 0.05, 200)
    ix = ak.Index(X)
    # poison the host-output staging with another call first
    ix.query(Q[::-1].copy(), 4, 4, 0.05, 99, al, sums=True)
    got = ix.query(Q, 4, 4, 0.05, 5, al, sums=True, max_rounds=3, batch_queries=2, timing=timing)
    ix.close()
    assert got["status"] == ak.AKNN_EMAXROUNDS
    ref = orc.query_br(X, Q, 4, 4, 5, al, want_sums=True, max_rounds=3)
    _eq(got, ref)


def test_sharded_sub_batches_with_round_cap(ak):
    X, Q = synth.small_instance(73, 3000, 96, q=5)
    al = orc.alpha_theory(3000, 0.05, 96)
    shards = [ak.Index(X[a:b], n_global=3000, offset=a) for a, b in ((0, 1000), (1000, 3000))]
    got = ak.query_multi(shards, Q, 3, 3, 0.05, 8, al, sums=True, max_rounds=2, batch_queries=2)
    for s in shards:
        s.close()
    assert got["status"] == ak.AKNN_EMAXROUNDS
    ref = orc.query_br(X, Q, 3, 3, 8, al, want_sums=True, max_rounds=2)
    _eq(got, ref)


def test_sharded_stats_equal_single_index(ak):
    """tile_draws / level_mma_tiles / draws of query_multi = the same query on one index."""
    # the cut at 3072 is a multiple of every tile width (32 points, 1024-arm filter CTAs,
    # 256-point tensor-core tiles), so both runs make the same dense-tile decisions
    X, Q = synth.small_instance(74, 6144, 256, q=40)
    al = orc.alpha_theory(6144, 0.05, 256)
    ix = ak.Index(X)
    one = ix.query(Q, 5, 5, 0.05, 3, al)
    s1 = ix.stats()
    ix.close()
    shards = [ak.Index(X[a:b], n_global=6144, offset=a) for a, b in ((0, 3072), (3072, 6144))]
    two = ak.query_multi(shards, Q, 5, 5, 0.05, 3, al)
    s2 = shards[0].stats()
    for s in shards:
        s.close()
    _eq(two, one, ("sets", "dhat", "counts", "evals", "draws", "rounds"))
    for key in ("draws", "exact_fallbacks", "tile_draws", "tile_blocks", "philox_blocks", "level_mma_tiles"):
        assert s1[key] == s2[key], key
    assert s1["tile_draws"] > 0


def test_bindings_validate_dimensions(ak):
    import torch
    X, Q = synth.small_instance(75, 500, 32, q=2)
    al = orc.alpha_theory(500, 0.05, 32)
    ix = ak.Index(X)
    with pytest.raises(ak.AknnError):
        ix.query_device(torch.zeros((2, 31), dtype=torch.uint8, device="cuda"), 3, 3, 0.05, 0, al)
    with pytest.raises(ak.AknnError):
        ix.query_device(torch.as_tensor(Q).cuda(), 3, 3, 0.05, 0, al[:-1])
    with pytest.raises(ak.AknnError):
        ix.query_device(torch.as_tensor(Q).cuda(), 3, 3, 0.05, 0,
                        torch.as_tensor(al[:-1]).cuda())
    with pytest.raises(ak.AknnError):
        ix.exact(np.zeros((2, 33), np.uint8), 3)
    with pytest.raises(ak.AknnError):
        ix.query(Q, 3, 3, 0.05, 0, al, batch_queries=-1)
    sh = [ak.Index(X[:250], n_global=500, offset=0), ak.Index(X[250:], n_global=500, offset=250)]
    with pytest.raises(ak.AknnError):
        ak.query_multi(sh, np.zeros((2, 30), np.uint8), 3, 3, 0.05, 0, al)
    with pytest.raises(ak.AknnError):
        ak.query_multi(sh, Q, 3, 3, 0.05, 0, al[:10])
    for s in sh:
        s.close()
    ix.close()


def test_build_rejects_key_overflow(ak):
    """aknn.h domain: the composite rank key must fit 63 bits at build time."""
    # 33025 odd: bit_length(65025 * 2^15 * 33025) = 46, plus 18 bits of id for n > 2^17: 64 > 63
    X = np.zeros(((1 << 17) + 1, 33025), np.uint8)  # calloc: never touched
    with pytest.raises(ak.AknnError) as e:
        ak.Index(X)
    assert e.value.status == ak.AKNN_EINVAL


def test_exact_on_other_stream_after_deferred_query(ak):
    """The row norms computed by a deferred async query are waited for by an exact
    pass on another stream (event ordering)."""
    import torch
    X, Q = synth.small_instance(76, 30000, 512, q=64)
    al = orc.alpha_theory(30000, 0.05, 512)
    ix = ak.Index(X)
    dQ = torch.as_tensor(Q).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        ix.query_device(dQ, 5, 5, 0.05, 0, torch.as_tensor(al).cuda(), stream=s1)
    idx, dist = ix.exact_device(dQ, 5, stream=s2)
    s2.synchronize()
    s1.synchronize()
    ridx, rdist = orc.bruteforce(X, Q, 5)
    assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(dist.cpu().numpy(), rdist)
    ix.close()
