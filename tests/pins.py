"""Independent closed forms and golden-file readers used as parity pins.

Nothing here calls the oracle or the CUDA path."""
from __future__ import annotations

import os
from math import isqrt

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name: str) -> list[list[str]]:
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            rows.append(line.split())
    return rows


def paper_windows() -> list[tuple[int, int, int]]:
    """(lo, hi, #E in (lo, hi]) from Table 1."""
    return [(int(r[1]), int(r[2]), int(r[3])) for r in golden("paper_values.txt")
            if r[0] == "window"]


def _mobius_upto(n: int) -> np.ndarray:
    mu = np.ones(n + 1, dtype=np.int64)
    is_p = np.ones(n + 1, dtype=bool)
    is_p[:2] = False
    for p in range(2, isqrt(n) + 1):
        if is_p[p]:
            is_p[p * p::p] = False
    for p in np.flatnonzero(is_p):
        p = int(p)
        mu[p::p] *= -1
        if p * p <= n:
            mu[p * p::p * p] = 0
    return mu


def pi_D_closed_form(x: int) -> int:
    """#{d <= x : d = 5 mod 8, d squarefree} by
    Moebius inversion over odd m (m^2 = 1 mod 8 so d/m^2 = 5 mod 8):
    sum_{m odd} mu(m) * #{n <= x/m^2 : n = 5 mod 8}."""
    M = isqrt(x)
    mu = _mobius_upto(M)
    tot = 0
    for m in range(1, M + 1, 2):
        if mu[m]:
            tot += int(mu[m]) * ((x // (m * m) + 3) // 8)
    return tot


def prime_mask(lo: int, hi: int) -> np.ndarray:
    """is_prime[k] for the integers lo + k, lo <= lo + k <= hi, by a plain
    segmented Eratosthenes (independent of the oracle and of the CUDA sieve)."""
    n = hi - lo + 1
    mask = np.ones(n, dtype=bool)
    r = isqrt(hi)
    small = np.ones(r + 1, dtype=bool)
    small[:2] = False
    for p in range(2, isqrt(r) + 1):
        if small[p]:
            small[p * p::p] = False
    for p in np.flatnonzero(small):
        p = int(p)
        start = max(p * p, ((lo + p - 1) // p) * p)
        mask[start - lo::p] = False
    for v in (0, 1):
        if lo <= v <= hi:
            mask[v - lo] = False
    return mask
