"""Multi-GPU orchestration: one process per GPU, torch.distributed for plumbing.

The path shards with no data exchange: every d is independent (SURVEY.md
8(e)).  Each rank walks a contiguous shard of (lo, hi] into per-checkpoint
bucket counts on its own GPU (``eis_count_buckets_dev``); the only exchange is
ONE all-reduce (sum) of the 2*n int64 buckets over NCCL (NVLink/NVSwitch),
after which the inclusive prefix runs in the library's prefix kernel
(``eis_prefix_dev``).  Results are bit-identical for any number of ranks.

The host logic (``shard_bounds``, ``allreduce_buckets``) is exercised by CPU
``gloo`` tests with world_size 2; the counting itself always runs in the
CUDA library.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import classify_range, count_buckets_dev, prefix_dev
from . import shard_bounds as _shard_bounds


# The AUTO path's crossover, which the "auto" split's cost model uses (the
# library's option "crossover"; the model itself is in eis_shard_bounds).
AUTO_CROSSOVER = 750_000_000


def shard_bounds(lo: int, hi: int, world: int, rank: int, balance: str = "flat") -> tuple[int, int]:
    """Contiguous shard (a, b] of (lo, hi] for ``rank``; the
    split is the library's (``eis_shard_bounds``, host-only).

    balance="flat": equal widths (per-d cost is flat inside a window near a
    fixed scale).  balance="prefix": equal cost for a prefix (0, X] where the
    per-d cost grows like d^(1/4), so the cumulative cost grows like x^(5/4):
    cut points x_g = X (g/G)^(4/5).  balance="auto": equal cost under the
    measured cost of the AUTO path (HALF ~ d^(1/2) below the crossover, BSGS
    ~ d^0.238 above), integrated numerically over (lo, hi].  Interior
    boundaries are multiples of 8 (never = 5 mod 8), so no candidate is split.
    """
    return _shard_bounds(lo, hi, world, rank, balance)


def allreduce_buckets(buckets: torch.Tensor, group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """The path's one exchange step: sum the 2*n bucket counts over all ranks
    (NCCL over NVLink on GPUs; any backend works, the tests use gloo)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if buckets.is_cuda and dist.get_backend(group) == "gloo":
            # gloo (the CPU tests' and --share-gpu's backend) reduces host tensors
            h = buckets.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            buckets.copy_(h)
        else:
            dist.all_reduce(buckets, op=dist.ReduceOp.SUM, group=group)
    return buckets


def count_window_distributed(lo: int, x, group: Optional[dist.ProcessGroup] = None,
                             balance: str = "auto") -> tuple[np.ndarray, np.ndarray]:
    """cnt_D[i], cnt_E[i] over lo < d <= x[i], computed by all ranks of ``group``
    (one GPU each, the current CUDA device).  Every rank passes the same (lo, x)
    and receives the full result."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
    n = len(x)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    a, b = shard_bounds(lo, int(x[-1]), world, rank, balance)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    buckets = torch.zeros(2 * n, dtype=torch.int64, device=dev)
    count_buckets_dev(a, b, x, buckets, stream=stream)
    allreduce_buckets(buckets, group)
    prefix_dev(buckets, buckets, stream=stream)
    h = buckets.cpu().numpy().astype(np.uint64)
    return h[:n], h[n:]


def classify_range_distributed(lo: int, hi: int, group: Optional[dist.ProcessGroup] = None,
                               balance: str = "flat") -> tuple[int, int, np.ndarray]:
    """This rank's slice of classify_range(lo, hi) (disjoint
    slices, D2H, no collective).  Returns (a, b, flags): flags classify every
    candidate d in (a, b]; the slices of ranks 0..world-1 concatenated in rank
    order equal classify_range(lo, hi)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    a, b = shard_bounds(max(lo, 1) - 1, hi, world, rank, balance)
    return a, b, classify_range(a + 1, b)
