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

from . import count_buckets_dev, prefix_dev


# Measured per-d device cost of the default (AUTO) path on one B200:
# HALF below the crossover, rate ~ 2.68e8 (1e10/d)^(1/2) d/s; BSGS at and above
# it, rate ~ 4.42e8 (1e10/d)^0.228 d/s.  Only the shape matters for splitting.
AUTO_CROSSOVER = 1_450_000_000


def auto_cost_density(d: np.ndarray) -> np.ndarray:
    """Relative device time per candidate at d under EIS_MODE_AUTO."""
    d = np.maximum(np.asarray(d, dtype=np.float64), 1.0)
    half = (d / 1e10) ** 0.5 / 2.68e8
    bsgs = (d / 1e10) ** 0.228 / 4.42e8
    return np.where(d < AUTO_CROSSOVER, half, bsgs)


def shard_bounds(lo: int, hi: int, world: int, rank: int, balance: str = "flat") -> tuple[int, int]:
    """Contiguous shard (a, b] of (lo, hi] for ``rank``.

    balance="flat": equal widths (per-d cost is flat inside a window near a
    fixed scale).  balance="prefix": equal cost for a prefix (0, X] where the
    per-d cost grows like d^(1/4), so the cumulative cost grows like x^(5/4):
    cut points x_g = X (g/G)^(4/5).  balance="auto": equal cost under the
    measured cost of the AUTO path (HALF ~ d^(1/2) below 1.45e9, BSGS ~ d^0.228
    above), integrated numerically over (lo, hi].  Boundaries are rounded to
    multiples of 8 (never = 5 mod 8), so no candidate is split.
    """
    if world <= 1:
        return lo, hi
    cum = None
    if balance == "auto":
        xs = np.linspace(lo, hi, 4097)
        c = auto_cost_density(np.maximum(xs, 1.0))
        cum = np.concatenate([[0.0], np.cumsum(0.5 * (c[1:] + c[:-1]) * np.diff(xs))])
        cum /= cum[-1]

    def cut(g: int) -> int:
        if g <= 0:
            return lo
        if g >= world:
            return hi
        if balance == "prefix":
            v = lo + int((hi - lo) * (g / world) ** 0.8)
        elif balance == "auto":
            v = int(np.interp(g / world, cum, xs))
        else:
            v = lo + (hi - lo) * g // world
        return min(hi, max(lo, v - v % 8))

    return cut(rank), cut(rank + 1)


def allreduce_buckets(buckets: torch.Tensor, group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """The path's one exchange step: sum the 2*n bucket counts over all ranks
    (NCCL over NVLink on GPUs; any backend works, the tests use gloo)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
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
