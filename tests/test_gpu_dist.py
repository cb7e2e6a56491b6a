"""GPU parity of the device-resident and multi-rank path (SURVEY.md 8(a) row a6,
8(e)): the bench's timed region ``count_buckets_dev -> all-reduce -> prefix_dev``,
``classify_range_dev``, ``count_window_distributed`` and its flag counterpart
``classify_range_distributed`` (world size 1, and 2 ranks sharing one GPU over
gloo), the library's own NCCL communicator (``eis_count_window_comm``), and the
C example that drives it -- each against the CPU oracle, bit-exact.

Two ranks share cuda:0 here (the box has one GPU).  Their kernels never wait on
one another: each rank walks its own shard and the one exchange is a host
(gloo) all-reduce, so this tests the orchestration, not a measurement.
"""
import json
import os
import socket
import subprocess

import numpy as np
import pytest
import torch

import paper_2507_06579_b200 as eis
from oracle import c_oracle
from paper_2507_06579_b200.dist import classify_range_distributed, count_window_distributed

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# A window that spans the AUTO crossover (moved down to 600,005 here), many
# sieve chunks and, with segment_log2 = 18, several segments; ragged ends.
LO = 123_457
X = [300_000, 600_000, 600_005, 600_013, 1_000_003, 2_345_677]


@pytest.fixture(autouse=True)
def _small_crossover_many_segments():
    from paper_2507_06579_b200 import _build

    _build.build()
    eis.init(0)
    old = {k: eis.get_option(k) for k in ("crossover", "segment_log2", "mode")}
    eis.set_option("crossover", 600_005)
    eis.set_option("segment_log2", 18)
    eis.set_option("mode", eis.MODE_AUTO)
    yield
    for k, v in old.items():
        eis.set_option(k, v)


def _oracle_counts(lo, x):
    oD, oE = c_oracle.count_window(lo, x)
    return oD.astype(np.uint64), oE.astype(np.uint64)


def test_count_buckets_dev_then_prefix_dev():
    """The bench's timed region on a non-default stream: buckets of two
    disjoint shards accumulated into one device array, then the prefix kernel."""
    n = len(X)
    oD, oE = _oracle_counts(LO, X)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    buckets = torch.zeros(2 * n, dtype=torch.int64, device=dev)
    out = torch.empty_like(buckets)
    stream.wait_stream(torch.cuda.current_stream(dev))       # the zero-fill
    with torch.cuda.stream(stream):
        cut = 1_000_000                                      # a multiple of 8
        eis.count_buckets_dev(LO, cut, X, buckets, stream=stream)
        eis.count_buckets_dev(cut, X[-1], X, buckets, stream=stream)
        eis.prefix_dev(buckets, out, stream=stream)
    stream.synchronize()
    got = out.cpu().numpy().astype(np.uint64)
    assert np.array_equal(got[:n], oD) and np.array_equal(got[n:], oE)
    # the raw buckets are the differences of the counts
    b = buckets.cpu().numpy().astype(np.int64)
    assert np.array_equal(np.cumsum(b[:n]), oD.astype(np.int64))
    # in place (out == buckets), as the bench does
    eis.prefix_dev(buckets, buckets)
    torch.cuda.synchronize()
    assert np.array_equal(buckets.cpu().numpy().astype(np.uint64), got)
    # d beyond x[n-1] are not counted
    z = torch.zeros(2 * n, dtype=torch.int64, device=dev)
    eis.count_buckets_dev(X[-1], X[-1] + 10_000, X, z)
    torch.cuda.synchronize()
    assert int(z.abs().sum()) == 0


def test_classify_range_dev_matches_oracle():
    lo, hi = LO, X[-1]
    n = eis.num_candidates(lo, hi)
    out = torch.full((n + 7,), 0xEE, dtype=torch.uint8, device="cuda:0")
    eis.classify_range_dev(lo, hi, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    want = c_oracle.classify_range(lo, hi)
    assert np.array_equal(got[:n], want)
    assert np.all(got[n:] == 0xEE)                          # nothing written past the range
    with pytest.raises(eis.EisError):
        eis.classify_range_dev(lo, hi, out[: n - 1])         # short buffer


@pytest.mark.parametrize("balance", ["flat", "prefix", "auto"])
def test_count_window_distributed_world1(balance):
    oD, oE = _oracle_counts(LO, X)
    cD, cE = count_window_distributed(LO, X, balance=balance)
    assert np.array_equal(cD, oD) and np.array_equal(cE, oE)
    a, b, f = classify_range_distributed(LO, X[-1], balance=balance)
    assert (a, b) == (LO - 1, X[-1])
    assert np.array_equal(f, c_oracle.classify_range(LO, X[-1]))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eis.init(0)
        eis.set_option("crossover", 600_005)
        eis.set_option("segment_log2", 18)
        res = {}
        for balance in ("flat", "prefix", "auto"):
            cD, cE = count_window_distributed(LO, X, balance=balance)
            a, b, f = classify_range_distributed(LO, X[-1], balance=balance)
            res[balance] = (cD.tolist(), cE.tolist(), a, b, f.tobytes())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_ranks_share_one_gpu_over_gloo():
    """world size 2 (gloo, both ranks on cuda:0): every rank receives counts
    equal to the oracle's for each split; the flag slices are disjoint and
    concatenate to the oracle's flags of the whole range."""
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    oD, oE = _oracle_counts(LO, X)
    want = c_oracle.classify_range(LO, X[-1])
    for balance in ("flat", "prefix", "auto"):
        parts = []
        for r in range(world):
            cD, cE, a, b, fb = res[r][balance]
            assert cD == oD.tolist() and cE == oE.tolist(), (balance, r)
            parts.append((a, b, np.frombuffer(fb, dtype=np.uint8)))
        assert parts[0][0] == LO - 1 and parts[-1][1] == X[-1] and parts[0][1] == parts[1][0]
        assert parts[0][1] > parts[0][0] and parts[1][1] > parts[1][0]   # both ranks worked
        assert np.array_equal(np.concatenate([f for _, _, f in parts]), want), balance


def test_library_communicator_world1():
    """eis_comm_unique_id / eis_comm_init / eis_count_window_comm: the C ABI's
    own NCCL path (all-reduce on the library's stream) at world size 1."""
    uid = eis.comm_unique_id()
    assert len(uid) == 128
    eis.comm_init(uid, 1, 0)
    try:
        cD, cE = eis.count_window_comm(LO, X)
        oD, oE = _oracle_counts(LO, X)
        assert np.array_equal(cD, oD) and np.array_equal(cE, oE)
    finally:
        eis.comm_finalize()
    # without a communicator it is eis_count_window
    cD, cE = eis.count_window_comm(LO, X)
    assert np.array_equal(cD, oD) and np.array_equal(cE, oE)


def test_c_example_count_box(tmp_path):
    """examples/count_box.c: a C program that counts over the whole box through
    eis_comm_* (world size 1 here), against the oracle."""
    exe = str(tmp_path / "count_box")
    pkg = os.path.join(ROOT, "paper_2507_06579_b200")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "count_box.c"), "-L", pkg, "-leis",
                           f"-Wl,-rpath,{pkg}", "-o", exe])
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
               EIS_ID_FILE=str(tmp_path / "id"))
    x = [10**5, 10**6, 3_000_001]
    out = subprocess.run([exe, "0", *map(str, x)], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    oD, oE = _oracle_counts(0, x)
    assert line["D"] == oD.tolist() and line["E"] == oE.tolist()
    assert line["E"][0] == 2942                              # pi_E(1e5), SURVEY.md 8(c)
