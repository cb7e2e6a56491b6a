"""Seeded synthetic workloads shared by the tests, smoke() and bench.py.

Holds NONE of the method's arithmetic: only ranges, checkpoint lists and
seeded samplers of candidate integers d = 5 (mod 8).  Whether a candidate is
squarefree, and its residue, is decided separately by the oracle and by the
CUDA path.

The workloads are the paper's own: every d in a range ("We
computed pi_E(x) for x <= 10^11"; Table 1 windows of length 10^8, l.416-464),
as configured in BASELINE.json ``configs``:

  C1  all d <= 1e5                       checkpoints 1e3, 1e4, 1e5
  C2  all d <= 1e8                       checkpoints every 1e7
  C3  all d <= 1e9                       checkpoints every 1e7
  C4  window (1e11 - 1e9, 1e11]          checkpoints every 1e8
  C5  all d <= 1e11 (8 GPUs)             checkpoints every 1e7
  METRIC window (9e9, 1e10] "at d ~ 1e10" split in 8 slabs of 1.25e8
"""
from __future__ import annotations

import numpy as np

SEED = 20250709

CONFIGS = {
    "C1": dict(lo=0, hi=10**5, x=[10**3, 10**4, 10**5]),
    "C2": dict(lo=0, hi=10**8, x=[k * 10**7 for k in range(1, 11)]),
    "C3": dict(lo=0, hi=10**9, x=[k * 10**7 for k in range(1, 101)]),
    "C4": dict(lo=10**11 - 10**9, hi=10**11, x=[10**11 - 10**9 + k * 10**8 for k in range(1, 11)]),
    "C5": dict(lo=0, hi=10**11, x=[k * 10**7 for k in range(1, 10**4 + 1)]),
}

# Metric workload: the window (9e9, 1e10], cut into 8 slabs of
# width 1.25e8; rank r of an N-GPU job owns slab r, counted down from 1e10, so
# N=1 is (9.875e9, 1e10] (which contains Table 1's window (9.9e9, 1e10]) and
# N=8 is the whole window.  Per-GPU work is fixed (weak scaling).
METRIC_TOP = 10**10
METRIC_SLAB = 125_000_000
METRIC_STRIDE = 10**7


def metric_slab(rank: int) -> tuple[int, int]:
    """(lo, hi] of slab ``rank``."""
    hi = METRIC_TOP - rank * METRIC_SLAB
    return hi - METRIC_SLAB, hi


def metric_window(n_ranks: int) -> tuple[int, int]:
    return METRIC_TOP - n_ranks * METRIC_SLAB, METRIC_TOP


def metric_checkpoints(n_ranks: int) -> list[int]:
    """Checkpoints every 1e7 inside the job's window, always including the top
    and the Table 1 boundary 9.9e9 (both multiples of 1e7)."""
    lo, hi = metric_window(n_ranks)
    first = (lo // METRIC_STRIDE + 1) * METRIC_STRIDE
    return list(range(first, hi + 1, METRIC_STRIDE))


def candidates(lo: int, hi: int) -> np.ndarray:
    """All integers d = 5 mod 8 with lo <= d <= hi (uint64)."""
    first = lo + ((5 - lo) % 8)
    if first > hi:
        return np.zeros(0, dtype=np.uint64)
    return np.arange(first, hi + 1, 8, dtype=np.uint64)


def sample_candidates(lo: int, hi: int, n: int, seed: int = SEED) -> np.ndarray:
    """n distinct candidates d = 5 mod 8 in [lo, hi], uniform, seeded, sorted."""
    first = lo + ((5 - lo) % 8)
    m = 0 if first > hi else (hi - first) // 8 + 1
    rng = np.random.default_rng(seed)
    n = min(n, m)
    idx = rng.choice(m, size=n, replace=False) if m < 2**62 else rng.integers(0, m, n)
    return np.sort(np.uint64(first) + np.uint64(8) * idx.astype(np.uint64))
