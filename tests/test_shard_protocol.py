"""The N > 1 exchange on CPUs (-m "not gpu").

The point-sharded round sends, per shard and query, the local top-(k+h) arms
plus the minimum-L arm of the rest, all-gathers them, and merges them the same
way on every shard.  Here the library's host reference of that protocol
(aknn_shard_summary_host / aknn_shard_merge_host, the same records and tie
rules as k_select_local / k_merge) is run on arm states taken from the ORACLE
mid-run, split into shards, exchanged with torch.distributed (gloo, world
size 2 -- and in-process for larger worlds), and compared with the oracle's own
round quantities on the unsplit state (orc_round_step: R2-R4)."""
import os
import socket

import numpy as np
import pytest

import oracle.oracle as orc
import synth


def _lvl(T, d):
    T = np.asarray(T)
    out = np.zeros(T.shape, np.uint8)
    ex = T == d
    out[ex] = 0xFF
    out[~ex] = np.log2(T[~ex]).astype(np.uint8)
    assert np.all((1 << out[~ex].astype(np.int64)) == T[~ex])
    return out


def _states(seed, n, d, k, h, rounds, alpha, q=2):
    """Oracle arm states (S, T) of q queries after `rounds` evaluations."""
    X, Q = synth.small_instance(seed, n, d, q=q)
    r = orc.query_br(X, Q, k, h, 5, alpha, max_rounds=rounds, want_sums=True)
    return r["sums"], r["counts"]


def _expect(S, T, d, k, h, alpha):
    return orc.round_step(S, T, d, k, h, alpha, want_active=False)


def _merge_and_check(ak, recs_by_shard, S, T, n, d, k, h, alpha):
    m = ak.shard_merge_host(np.concatenate(recs_by_shard), len(recs_by_shard), n, d, k, h, alpha)
    e = _expect(S, T, d, k, h, alpha)
    kh = k + h
    assert m["sets"].tolist() == e["order"][:kh].tolist()
    assert m["stop"] == e["stop"]
    assert (m["d1"], m["d2"]) == (e["d1"], e["d2"])
    assert m["A"] == e["A"] and m["B"] == e["B"]  # same fp64 bits (one rounding each)
    a_d2 = 0.0 if T[e["d2"]] == d else alpha[T[e["d2"]]]
    assert m["alpha_d2"] == a_d2
    dh = S[e["order"][:kh]] / (T[e["order"][:kh]] * 65025.0)
    assert np.array_equal(m["dhat"], dh)


@pytest.fixture(scope="module")
def ak():
    import __graft_entry__
    __graft_entry__._load_builder().build()
    import paper_1902_09465_b200 as m
    return m


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("rounds", [1, 3, 6])
def test_in_process_shards_match_unsplit_round(ak, world, rounds):
    n, d, k, h = 1200, 96, 5, 7
    al = orc.alpha_experimental(n, 0.05, d, 0.05)
    Ss, Ts = _states(41 + rounds, n, d, k, h, rounds, al)
    bounds = np.linspace(0, n, world + 1).astype(int)
    for S, T in zip(Ss, Ts):
        lv = _lvl(T, d)
        recs = [ak.shard_summary_host(S[a:b].astype(np.int32), lv[a:b], a, n, d, k, h, al)
                for a, b in zip(bounds[:-1], bounds[1:])]
        _merge_and_check(ak, recs, S, T, n, d, k, h, al)


def test_uneven_shards_and_h0(ak):
    n, d, k, h = 900, 40, 6, 0
    al = orc.alpha_theory(n, 0.05, d)
    Ss, Ts = _states(7, n, d, k, h, 4, al)
    bounds = [0, 13, 400, 401 + 50, n]
    for S, T in zip(Ss, Ts):
        lv = _lvl(T, d)
        recs = [ak.shard_summary_host(S[a:b].astype(np.int32), lv[a:b], a, n, d, k, h, al)
                for a, b in zip(bounds[:-1], bounds[1:])]
        _merge_and_check(ak, recs, S, T, n, d, k, h, al)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1902_09465_b200 as ak
        n, d, k, h = 2000, 64, 8, 8
        al = orc.alpha_experimental(n, 0.05, d, 0.1)
        Ss, Ts = _states(99, n, d, k, h, 5, al, q=3)
        bounds = np.linspace(0, n, world + 1).astype(int)
        a, b = bounds[rank], bounds[rank + 1]
        outs = []
        for S, T in zip(Ss, Ts):
            lv = _lvl(T, d)
            mine = torch.from_numpy(
                ak.shard_summary_host(S[a:b].astype(np.int32), lv[a:b], a, n, d, k, h, al))
            got = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(got, mine)  # the exchange step (NCCL allgather on the GPU path)
            m = ak.shard_merge_host(torch.cat(got).numpy(), world, n, d, k, h, al)
            outs.append((m["sets"].tolist(), m["stop"], m["d1"], m["d2"], m["A"], m["B"]))
            _merge_and_check(ak, [g.numpy() for g in got], S, T, n, d, k, h, al)
        result_q.put((rank, outs))
    except Exception as e:  # surface the failure to the parent
        result_q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_matches_oracle(ak):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(not isinstance(v, str) for v in res.values()), res
    # both ranks reached the identical global decision for every query
    assert res[0] == res[1]
