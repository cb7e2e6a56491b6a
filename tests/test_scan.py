"""Checkpointed scan with resume (paper_2507_06579_b200/scan.py): host logic.

The counting backend is injected.  The CPU tests drive it with the oracle's
per-d residues and an independent prime sieve (tests only; the product's scan
counts on the GPU), and check that:
- an interrupted and resumed scan writes byte-identical CSV;
- a torn last line is dropped;
- a fingerprint mismatch is rejected;
- resuming a finished scan is a no-op.
The GPU test runs the same contract through the CUDA path.
"""
import os

import numpy as np
import pytest

from oracle import c_oracle
from paper_2507_06579_b200.scan import HEADER, fingerprint, scan
from pins import prime_mask


def oracle_rows(lo, x):
    """count_fn over (lo, x_i]: rows D, E, T1, DP, EP from the oracle."""
    x = np.asarray(x, dtype=np.int64)
    hi = int(x[-1])
    f = c_oracle.classify_range(lo + 1, hi)
    first = (lo + 1) + (5 - (lo + 1)) % 8
    d = first + 8 * np.arange(f.size, dtype=np.int64)
    pm = prime_mask(lo + 1, hi)[d - (lo + 1)] if f.size else np.zeros(0, bool)
    out = {k: np.zeros(len(x), dtype=np.uint64) for k in ("D", "E", "T1", "DP", "EP")}
    for i, xi in enumerate(x):
        m = d <= xi
        inD = m & (f != c_oracle.NOT_IN_D)
        out["D"][i] = inD.sum()
        out["E"][i] = (m & (f == 0)).sum()
        out["T1"][i] = (m & (f == 1)).sum()
        out["DP"][i] = (inD & pm).sum()
        out["EP"][i] = (m & (f == 0) & pm).sum()
    return out


def test_resume_is_byte_identical(tmp_path):
    full, part = tmp_path / "full.csv", tmp_path / "part.csv"
    n = scan(0, 200_000, 5_000, str(full), chunk=7, count_fn=oracle_rows)
    assert n == 40
    scan(0, 200_000, 5_000, str(part), chunk=7, count_fn=oracle_rows, max_chunks=2)
    scan(0, 200_000, 5_000, str(part), chunk=7, count_fn=oracle_rows, max_chunks=1)
    scan(0, 200_000, 5_000, str(part), chunk=7, count_fn=oracle_rows)
    assert full.read_bytes() == part.read_bytes()
    lines = full.read_text().splitlines()
    assert lines[0] == fingerprint(0, 200_000, 5_000, 7) and lines[1] == HEADER
    last = [int(v) for v in lines[-1].split(",")]
    assert last[0] == 200_000
    D, E = c_oracle.count_window(0, [200_000])
    assert last[1] == int(D[0]) and last[2] == int(E[0])
    # counter invariants at every checkpoint: E <= D, EP <= E, DP <= D, T1 <= D - E
    for ln in lines[2:]:
        x, d, e, t1, dp, ep = (int(v) for v in ln.split(","))
        assert e <= d and ep <= e and dp <= d and t1 <= d - e


def test_torn_tail_fingerprint_and_noop(tmp_path):
    p = tmp_path / "s.csv"
    scan(10_000, 50_000, 1_000, str(p), chunk=5, count_fn=oracle_rows, max_chunks=3)
    good = p.read_text()
    with open(p, "a") as f:                     # an interrupted write
        f.write("26000,12")
    n = scan(10_000, 50_000, 1_000, str(p), chunk=5, count_fn=oracle_rows)
    assert n == 40
    ref = tmp_path / "ref.csv"
    scan(10_000, 50_000, 1_000, str(ref), chunk=5, count_fn=oracle_rows)
    assert p.read_bytes() == ref.read_bytes() and p.read_text().startswith(good)
    calls = []
    n2 = scan(10_000, 50_000, 1_000, str(p), chunk=5,
              count_fn=lambda lo, x: calls.append(1) or oracle_rows(lo, x))
    assert n2 == 40 and not calls                # finished: no-op
    with pytest.raises(ValueError):
        scan(10_000, 50_000, 2_000, str(p), chunk=5, count_fn=oracle_rows)


def test_ragged_last_checkpoint(tmp_path):
    p = tmp_path / "r.csv"
    n = scan(0, 10_007, 1_000, str(p), chunk=4, count_fn=oracle_rows)
    xs = [int(ln.split(",")[0]) for ln in p.read_text().splitlines()[2:]]
    assert n == 11 and xs[-1] == 10_007 and xs[:-1] == list(range(1_000, 10_001, 1_000))


@pytest.mark.gpu
def test_scan_through_the_cuda_path_matches_oracle_backend(tmp_path):
    import paper_2507_06579_b200 as eis
    eis.init(0)
    g, o = tmp_path / "gpu.csv", tmp_path / "oracle.csv"
    scan(0, 400_000, 10_000, str(g), chunk=9, max_chunks=2)
    scan(0, 400_000, 10_000, str(g), chunk=9)
    scan(0, 400_000, 10_000, str(o), chunk=9, count_fn=oracle_rows)
    assert g.read_bytes() == o.read_bytes()
