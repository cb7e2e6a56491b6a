"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY (pure Python twin of eis_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It shares nothing with
the CUDA path (paper_2507_06579_b200/) and never calls it.

This is the plain definition of the classified quantity, written with Python
big integers for small cases (d up to ~1e7 in seconds per thousand d):

* PAPER.md l.52-55 (Sec. 1): for squarefree d = 5 mod 8, O_K = Z[w] with
  w = (1+sqrt d)/2, and eps_d = (x0 + y0 sqrt d)/2 is the fundamental unit.
* D = {d > 0 : d = 5 mod 8, d squarefree};
  E = {d in D : eps_d = 1 mod 2 O_K}.
* pi_E(x), pi_D(x) count d in E (resp. D) with d <= x.
* (O_K/2O_K)^* = F_4^* = Z/3; the residue t of eps_d is
  its discrete log, and t == 0 iff d in E.

eps_d is computed from the regular continued fraction of w (the standard
fact that the convergent p/q just before the first return of the complete
quotient denominator to Q = 2 gives the fundamental unit p - q*conj(w));
every result is certified by the exact norm identity x0^2 - d y0^2 = +-4.
The tests pin the fundamental-unit claim independently by brute force
(tests/test_oracle.py).
"""
from __future__ import annotations

from math import isqrt

# (a mod 2, b mod 2) of a*1 + b*w  ->  discrete log in F_4^* (
# the labelling 1 -> 0, w -> 1, w^2 = w+1 -> 2 is one fixed choice).
DLOG = {(1, 0): 0, (0, 1): 1, (1, 1): 2}

NOT_IN_D = 0xFF


def is_squarefree(d: int) -> bool:
    """trial division by every odd m >= 3 with m^2 <= d."""
    if d <= 0 or d % 4 == 0:
        return False
    m = 3
    while m * m <= d:
        if d % (m * m) == 0:
            return False
        m += 2
    return True


def in_D(d: int) -> bool:
    """d in D iff d = 5 mod 8 and squarefree."""
    return d % 8 == 5 and is_squarefree(d)


def fundamental_unit(d: int) -> tuple[int, int, int, int]:
    """eps_d = (x0 + y0 sqrt d)/2 via the continued fraction of (1+sqrt d)/2.

    Returns (x0, y0, norm, period) with norm = x0^2 - d y0^2 in {+4, -4}
    (asserted exactly) and period the CF period length.
    """
    if d % 4 != 1 or isqrt(d) ** 2 == d:
        raise ValueError("need non-square d = 1 mod 4")
    s = isqrt(d)
    P, Q = 1, 2                      # complete quotient (P + sqrt d)/Q = w
    p1, p2 = 1, 0                    # p_{k-1}, p_{k-2}
    q1, q2 = 0, 1                    # q_{k-1}, q_{k-2}
    k = 0
    while True:
        a = (P + s) // Q             # a_k = floor((P + sqrt d)/Q) for Q > 0
        p1, p2 = a * p1 + p2, p1
        q1, q2 = a * q1 + q2, q1
        P = a * Q - P
        num = d - P * P
        assert num % Q == 0
        Q = num // Q
        k += 1
        if Q == 2:                   # first return: end of the period
            break
    x0, y0 = 2 * p1 - q1, q1
    norm = x0 * x0 - d * y0 * y0
    assert norm in (4, -4), (d, norm)
    return x0, y0, norm, k


def residue(d: int) -> int:
    """t(eps_d) in Z/3 for d in D: eps = (p-q)*1 + q*w."""
    if not in_D(d):
        raise ValueError(f"{d} not in D")
    x0, y0, _, _ = fundamental_unit(d)
    # x0 = 2p - q, y0 = q  =>  p - q = (x0 - y0)/2
    return DLOG[(((x0 - y0) // 2) % 2, y0 % 2)]


def classify_range(lo: int, hi: int) -> list[int]:
    """One entry per candidate d = first + 8i <= hi (first = least d >= lo,
    d = 5 mod 8): t(eps_d), or NOT_IN_D for non-squarefree d."""
    first = lo + ((5 - lo) % 8)
    out = []
    d = first
    while d <= hi:
        out.append(residue(d) if is_squarefree(d) else NOT_IN_D)
        d += 8
    return out


def count(xs: list[int], lo: int = 0) -> tuple[list[int], list[int]]:
    """(cnt_D, cnt_E) over lo < d <= x for each checkpoint x (ascending)."""
    cD, cE, outD, outE = 0, 0, [], []
    d = (lo + 1) + ((5 - (lo + 1)) % 8)
    for x in xs:
        while d <= x:
            if is_squarefree(d):
                cD += 1
                cE += residue(d) == 0
            d += 8
        outD.append(cD)
        outE.append(cE)
    return outD, outE
