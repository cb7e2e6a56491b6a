"""Pins for the CPU oracle against things other than itself (CPU only).

Each test names the passage or mathematical fact it pins.  A plausible slip in
the oracle (wrong convergent index, wrong x0 = 2p - q, transposed DLOG table,
off-by-one in the squarefree bound, wrong stop rule) fails at least one test:

* brute force: the smallest solution of x^2 - d y^2 = +-4 (definition of the
  fundamental unit) for every tiny d in D;
* Lemma 1.1 (1)<=>(2) by brute-force search for odd solutions
  of x^2 - d y^2 = 4;
* DLOG is a group homomorphism (O_K/2O_K)^* -> Z/3, checked
  on exact products in O_K;
* the paper's printed examples and textbook units;
* pi_D against the Moebius closed form;
* Table 1 prefix total pi_E(1e8) = 3,259,668 (slow, EIS_SLOW=1).
"""
import os
from math import isqrt

import numpy as np
import pytest

from oracle import c_oracle as C
from oracle import oracle as O

from pins import golden as _golden, pi_D_closed_form


def D_upto(n):
    return [d for d in range(5, n + 1, 8) if O.is_squarefree(d)]


# ----------------------------------------------------------------- brute force --
def _is_square(v: np.ndarray) -> np.ndarray:
    r = np.floor(np.sqrt(v.astype(np.float64))).astype(np.int64)
    ok = np.zeros(v.shape, dtype=bool)
    for dr in (-1, 0, 1):
        rr = r + dr
        ok |= (rr >= 0) & (rr * rr == v)
    return ok


@pytest.mark.parametrize("impl", ["py", "c"])
def test_fundamental_unit_brute_force(impl):
    """eps_d is the solution of x^2 - d y^2 = +-4 with the least y > 0
    (eps_d = (x0 + y0 sqrt d)/2 fundamental)."""
    Y = 400_000
    ys = np.arange(1, Y + 1, dtype=np.int64)
    unit = O.fundamental_unit if impl == "py" else C.fundamental_unit
    resolved = 0
    for d in D_upto(1000):
        x0, y0, norm, _ = unit(d)
        dy2 = d * ys * ys
        hit = _is_square(dy2 + 4) | _is_square(dy2 - 4)
        idx = np.flatnonzero(hit)
        if idx.size == 0:
            assert y0 > Y, d
            continue
        resolved += 1
        y = int(ys[idx[0]])
        assert y0 == y, (d, y0, y)
        cand = [isqrt(d * y * y + 4), isqrt(max(d * y * y - 4, 0))]
        assert x0 in cand and x0 * x0 - d * y0 * y0 in (4, -4), d
    assert resolved > 80


def test_lemma_1_1_odd_solutions():
    """PAPER.md l.77-86 Lemma (1)<=>(2): eps_d = 1 mod 2O_K iff x^2 - d y^2 = 4
    has no solution in odd x, y.  Brute force over odd y <= Y.  For t != 0 the
    first odd solution must be eps (norm +4) or eps^2 (y = x0 y0)."""
    Y = 1_000_001
    ys = np.arange(1, Y + 1, 2, dtype=np.int64)
    checked_pos = checked_neg = 0
    for d in D_upto(1200):
        t = O.residue(d)
        x0, y0, norm, _ = O.fundamental_unit(d)
        v = d * ys * ys + 4
        hit = _is_square(v)
        odd_x = hit & (np.floor(np.sqrt(v.astype(np.float64))).astype(np.int64) % 2 == 1)
        idx = np.flatnonzero(hit)
        if t == 0:
            assert idx.size == 0, (d, ys[idx[:3]])
            checked_neg += 1
        else:
            pred = y0 if norm == 4 else x0 * y0
            if pred <= Y:
                assert idx.size > 0 and int(ys[idx[0]]) == pred, (d, pred)
                assert odd_x[idx[0]]
                checked_pos += 1
    assert checked_pos > 30 and checked_neg > 10


def test_dlog_is_homomorphism():
    """(O_K/2O_K)^* = F_4^* = Z/3, multiplication becomes
    addition.  Exact products (a + b w)(c + e w) with w^2 = w + (d-1)/4 must map
    to sums of discrete logs under the oracle's DLOG table."""
    rng = np.random.default_rng(1)
    for d in (5, 13, 21, 101, 1901, 7053):
        k = (d - 1) // 4
        for _ in range(300):
            a, b, c, e = (int(v) for v in rng.integers(-1000, 1000, 4))
            if (a % 2, b % 2) == (0, 0) or (c % 2, e % 2) == (0, 0):
                continue
            # (a + b w)(c + e w) = ac + (ae + bc) w + be (w + k)
            x = a * c + b * e * k
            y = a * e + b * c + b * e
            t1 = O.DLOG[(a % 2, b % 2)]
            t2 = O.DLOG[(c % 2, e % 2)]
            assert O.DLOG[(x % 2, y % 2)] == (t1 + t2) % 3


def test_conjugation_negates_residue():
    """Frobenius on F_4 is the Galois conjugation: t(conj eps) = -t(eps)."""
    for d in D_upto(20000):
        x0, y0, _, _ = C.fundamental_unit(d)
        t = O.DLOG[(((x0 - y0) // 2) % 2, y0 % 2)]
        # conj eps = (x0 - y0 sqrt d)/2 = ((x0 + y0)/2) * 1 + (-y0) * w
        tc = O.DLOG[(((x0 + y0) // 2) % 2, (-y0) % 2)]
        assert (t + tc) % 3 == 0, d
        assert t == C.residue(d)


def test_paper_examples_and_textbook_units():
    for kind, d, cls in (r for r in _golden("paper_values.txt") if r[0] == "member"):
        assert (O.residue(int(d)) == 0) == (cls == "E")
        assert (C.residue(int(d)) == 0) == (cls == "E")
    for d, x0, y0, norm in _golden("textbook_units.txt"):
        d, x0, y0, norm = int(d), int(x0), int(y0), int(norm)
        assert O.fundamental_unit(d)[:3] == (x0, y0, norm)
        cx, cy, cs, _ = C.fundamental_unit(d)
        assert (cx, cy, 4 * cs) == (x0, y0, norm)


def test_non_squarefree_and_invalid_rejected():
    assert not O.is_squarefree(45) and not C.is_squarefree(45)     # 9 * 5
    assert not O.is_squarefree(5 * 49) and not C.is_squarefree(5 * 49)
    with pytest.raises(ValueError):
        O.residue(45)
    with pytest.raises(ValueError):
        C.residue(45)
    with pytest.raises(ValueError):
        C.residue(7)                                           # not 5 mod 8


# ---------------------------------------------------------- pi_D closed form --
def test_pi_D_matches_mobius_closed_form():
    xs = [10, 100, 1000, 12345, 10**5, 10**6]
    f = C.classify_range(0, 10**6)
    d = 5 + 8 * np.arange(f.size, dtype=np.int64)
    for x in xs:
        assert int(((f != C.NOT_IN_D) & (d <= x)).sum()) == pi_D_closed_form(x), x
    # D cap [0,100) = {5,13,21,29,37,53,61,69,77,85,93}
    assert [int(v) for v in d[(f != C.NOT_IN_D) & (d < 100)]] == [5, 13, 21, 29, 37, 53, 61,
                                                                    69, 77, 85, 93]


def test_c_and_python_oracles_agree():
    f = C.classify_range(0, 30000)
    g = O.classify_range(0, 30000)
    assert list(f) == g
    rng = np.random.default_rng(7)
    for d in rng.integers(10**6, 10**7, 60):
        d = int(d) - int(d) % 8 + 5
        if O.is_squarefree(d):
            assert O.residue(d) == C.residue(d)
            x, y, n, per = O.fundamental_unit(d)
            assert C.fundamental_unit(d) == (x, y, n // 4, per)


def test_count_window_consistent():
    xs = [1000, 5000, 20000]
    cD, cE = C.count_window(0, xs)
    pD, pE = O.count([1000, 5000, 20000])
    assert list(cD) == pD and list(cE) == pE
    cD2, cE2 = C.count_window(1000, [5000, 20000])
    assert list(cD2) == [pD[1] - pD[0], pD[2] - pD[0]]
    assert list(cE2) == [pE[1] - pE[0], pE[2] - pE[0]]


@pytest.mark.slow
def test_table1_prefix_total():
    """#E cap [0, 1e8] = 2,790,560+464,866+4,241+1."""
    rows = [r for r in _golden("paper_values.txt") if r[0] == "window"]
    lo, hi, want = (int(v) for v in rows[0][1:4])
    cD, cE = C.count_window(lo, [hi])
    assert int(cE[0]) == want
    assert int(cD[0]) == pi_D_closed_form(hi)


def test_count_window_boundaries_at_candidates():
    """eo_count_window at x = 5 (mod 8) (d <= x inclusive;
    windows exclude lo): 5 is the least d in D (t = 1, not in E) and 37 the
    least d in E (eps = 6 + sqrt 37); pi_D by the Moebius closed
    form at candidate-valued checkpoints and window ends."""
    cD, cE = C.count_window(0, [5, 37])
    assert list(cD) == [1, 5] and list(cE) == [0, 1]
    cD, cE = C.count_window(5, [37])                  # (5, 37]: 13, 21, 29, 37
    assert list(cD) == [4] and list(cE) == [1]
    cD, cE = C.count_window(37, [45])                 # (37, 45]: 45 = 9 * 5 is not in D
    assert list(cD) == [0] and list(cE) == [0]
    xs = [10_005, 99_997, 123_461, 200_005]            # all = 5 (mod 8)
    assert all(x % 8 == 5 for x in xs)
    cD, _ = C.count_window(0, xs)
    assert [int(v) for v in cD] == [pi_D_closed_form(x) for x in xs]
    lo = 10_005
    cD, _ = C.count_window(lo, xs[1:])
    assert [int(v) for v in cD] == [pi_D_closed_form(x) - pi_D_closed_form(lo) for x in xs[1:]]
