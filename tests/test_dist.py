"""Multi-GPU host logic on CPU: sharding and the one all-reduce, world_size 2 (gloo).

The path shards with no data exchange; the only collective is
the all-reduce of the 2n checkpoint buckets.  Here each rank fills the buckets
of its shard with the ORACLE (test infrastructure standing in for the CUDA
kernels, which need a GPU); the product functions under test are
``shard_bounds`` and ``allreduce_buckets``.  The combined counts must equal a
single-process count for any world size.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import c_oracle
import paper_2507_06579_b200 as eis
from paper_2507_06579_b200.dist import AUTO_CROSSOVER, allreduce_buckets, shard_bounds


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_buckets(a: int, b: int, x: np.ndarray) -> torch.Tensor:
    """Bucket counts of d in (a, b] (bucket(d) = least i with d <= x[i]) by the oracle."""
    n = len(x)
    out = np.zeros(2 * n, dtype=np.int64)
    top = min(b, int(x[-1]))
    if top > a:
        f = c_oracle.classify_range(a + 1, top)
        first = (a + 1) + (5 - (a + 1)) % 8
        d = first + 8 * np.arange(f.size, dtype=np.int64)
        bidx = np.searchsorted(x.astype(np.int64), d, side="left")
        np.add.at(out, bidx[f != c_oracle.NOT_IN_D], 1)
        np.add.at(out, n + bidx[f == 0], 1)
    return torch.from_numpy(out)


def _worker(rank, world, port, lo, x, balance, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = np.asarray(x, dtype=np.uint64)
        a, b = shard_bounds(lo, int(x[-1]), world, rank, balance)
        buckets = oracle_buckets(a, b, x)
        allreduce_buckets(buckets)
        q.put((rank, (a, b), buckets.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,balance", [(2, "flat"), (2, "prefix"), (3, "prefix"), (3, "auto")])
def test_sharded_allreduce_matches_single_process(world, balance):
    lo = 0 if balance == "prefix" else 123_457
    x = np.array([200_000, 350_001, 500_000, 777_777], dtype=np.uint64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lo, x, balance, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    shards = [r[1] for r in res]
    # shards are contiguous, disjoint and cover (lo, x[-1]]
    assert shards[0][0] == lo and shards[-1][1] == int(x[-1])
    for (a0, b0), (a1, b1) in zip(shards, shards[1:]):
        assert b0 == a1 and a0 <= b0 and b0 % 8 == 0
    # every rank holds the same reduced buckets, equal to the single-process ones
    want = oracle_buckets(lo, int(x[-1]), x).numpy()
    for _, _, got in res:
        assert np.array_equal(np.asarray(got), want)
    # prefix of the reduced buckets = counting functions
    n = len(x)
    cD, cE = c_oracle.count_window(lo, x)
    assert np.array_equal(np.cumsum(want[:n]), cD.astype(np.int64))
    assert np.array_equal(np.cumsum(want[n:]), cE.astype(np.int64))


def test_shard_bounds_properties():
    for world in (1, 2, 4, 8):
        for balance in ("flat", "prefix", "auto"):
            lo, hi = 9 * 10**9, 10**10
            cuts = [shard_bounds(lo, hi, world, r, balance) for r in range(world)]
            assert cuts[0][0] == lo and cuts[-1][1] == hi
            for (a0, b0), (a1, b1) in zip(cuts, cuts[1:]):
                assert b0 == a1 and b0 % 8 == 0
    # prefix balancing gives later (costlier per d) shards less width
    c = [shard_bounds(0, 10**9, 4, r, "prefix") for r in range(4)]
    widths = [b - a for a, b in c]
    assert widths == sorted(widths, reverse=True)


def auto_cost_density(d: np.ndarray) -> np.ndarray:
    """The AUTO path's measured per-d device cost, written out
    independently of the library's eis_shard_bounds: HALF below the crossover
    at 2.68e8 (1e10/d)^(1/2) d/s, BSGS above it at 5.0e8 (1e10/d)^0.224 d/s."""
    d = np.maximum(np.asarray(d, dtype=np.float64), 1.0)
    return np.where(d < AUTO_CROSSOVER, (d / 1e10) ** 0.5 / 2.68e8, (d / 1e10) ** 0.224 / 5.0e8)


def test_auto_balance_equalises_model_cost():
    """balance="auto" (the distributed default): on the C5 prefix (0, 1e11] each
    of 8 shards carries 1/8 of the modelled AUTO-path device time (HALF below
    the 7.5e8 crossover, BSGS above), to within the 8-aligned rounding."""
    X, G = 10**11, 8
    cuts = [shard_bounds(0, X, G, r, "auto") for r in range(G)]
    xs = np.linspace(1.0, X, 200001)
    c = auto_cost_density(xs)
    cum = np.concatenate([[0.0], np.cumsum(0.5 * (c[1:] + c[:-1]) * np.diff(xs))])
    share = [np.interp(b, xs, cum) - np.interp(a, xs, cum) for a, b in cuts]
    share = np.array(share) / cum[-1]
    assert np.all(np.abs(share - 1 / G) < 2e-3), share
    # the flat split would give the last shard ~1.3x the first's cost
    assert cuts[0][1] - cuts[0][0] > cuts[-1][1] - cuts[-1][0]


def test_shard_bounds_edges_and_errors():
    """eis_shard_bounds (host logic of the whole-box ABI): degenerate ranges,
    more ranks than candidates, and argument errors."""
    for balance in ("flat", "prefix", "auto"):
        assert shard_bounds(7, 7, 4, 2, balance) == (7, 7)
        assert shard_bounds(0, 100, 1, 0, balance) == (0, 100)
        cuts = [shard_bounds(100, 120, 8, r, balance) for r in range(8)]
        assert cuts[0][0] == 100 and cuts[-1][1] == 120
        assert all(b0 == a1 for (_, b0), (a1, _) in zip(cuts, cuts[1:]))
        assert sum(eis.num_candidates(a + 1, b) for a, b in cuts if b > a) == \
            eis.num_candidates(101, 120)
    for bad in [dict(world=0, rank=0), dict(world=2, rank=2), dict(world=2, rank=-1)]:
        with pytest.raises(eis.EisError):
            shard_bounds(0, 100, bad["world"], bad["rank"])
    with pytest.raises(eis.EisError):
        shard_bounds(10, 5, 2, 0)
    with pytest.raises(KeyError):
        shard_bounds(0, 100, 2, 0, "nope")


@pytest.mark.parametrize("lo,hi,world", [(0, 10**6, 2), (1, 999_999, 3), (5, 5, 2),
                                         (123_457, 9_876_543, 8), (10**10 - 10**6, 10**10, 4)])
def test_distributed_classify_slices_partition_the_range(lo, hi, world):
    """classify_range_distributed's slices (a+1 .. b of shard_bounds(lo-1, hi))
    are disjoint and, in rank order, hold exactly the candidates of [lo, hi]
    (per-d flags need no collective)."""
    for balance in ("flat", "prefix", "auto"):
        cuts = [shard_bounds(max(lo, 1) - 1, hi, world, r, balance) for r in range(world)]
        total = 0
        for r, (a, b) in enumerate(cuts):
            if r:
                assert a == cuts[r - 1][1]
            total += eis.num_candidates(a + 1, b) if b > a else 0
        assert total == eis.num_candidates(lo, hi)
