"""Checkpointed scan with resume.

``scan(lo, hi, stride, path)`` computes, for every checkpoint x = lo + k*stride
up to hi, the five counts of (lo, x]: D, E, T1 (t = 1), D cap P, E cap P
(Sec. 3, l.105-108 and Sec. 3.2, l.501-522).  Rows are appended to a
CSV one chunk at a time; each chunk is flushed and fsync'ed before the next
starts.  An interrupted scan resumes from its last complete row.  The output
is byte-identical to an uninterrupted run, because every row depends only on
(lo, x) and the format is fixed.

The first line is a fingerprint of the scan's parameters.  Resuming with other
parameters raises ``ValueError``.  Resuming a finished scan returns at once.

Host logic only.  Counting goes through ``count_fn(lo, x) -> dict of rows``,
which defaults to the library's ``count_window_ext`` (all arithmetic in the CUDA
kernels).
"""
from __future__ import annotations

import os
from typing import Callable, Optional

import numpy as np

ROWS = ("D", "E", "T1", "DP", "EP")
HEADER = "x,pi_D,pi_E,pi_T1,pi_DP,pi_EP"


def fingerprint(lo: int, hi: int, stride: int, chunk: int) -> str:
    return f"# eis-scan v1 lo={lo} hi={hi} stride={stride} chunk={chunk}"


def _checkpoints(lo: int, hi: int, stride: int) -> np.ndarray:
    xs = np.arange(lo + stride, hi + 1, stride, dtype=np.uint64)
    if len(xs) == 0 or int(xs[-1]) != hi:
        xs = np.append(xs, np.uint64(hi))
    return xs


def _read_state(path: str, fp: str) -> tuple[int, np.ndarray]:
    """(number of complete rows, last row's counts) of an existing scan file."""
    with open(path) as f:
        lines = f.read().split("\n")
    if not lines or lines[0] != fp:
        raise ValueError(f"{path}: fingerprint {lines[0] if lines else ''!r} != {fp!r}")
    if len(lines) < 2 or lines[1] != HEADER:
        raise ValueError(f"{path}: missing header")
    rows = [ln for ln in lines[2:] if ln]
    # a partial last line (interrupted write) has no trailing newline: drop it
    if rows and not lines[-1] == "":
        rows = rows[:-1]
    if not rows:
        return 0, np.zeros(len(ROWS), dtype=np.uint64)
    last = np.array([int(v) for v in rows[-1].split(",")[1:]], dtype=np.uint64)
    return len(rows), last


def scan(lo: int, hi: int, stride: int, path: str, *, chunk: int = 256,
         count_fn: Optional[Callable[[int, np.ndarray], dict]] = None,
         max_chunks: Optional[int] = None) -> int:
    """Run or resume the scan of (lo, hi] into ``path``; returns the number of rows
    now in the file.  ``max_chunks`` stops early (to emulate an interruption)."""
    if stride <= 0 or chunk <= 0 or lo >= hi:
        raise ValueError("need stride > 0, chunk > 0, lo < hi")
    if count_fn is None:
        from . import count_window_ext as count_fn   # the CUDA path
    fp = fingerprint(lo, hi, stride, chunk)
    xs = _checkpoints(lo, hi, stride)
    if os.path.exists(path):
        done, acc = _read_state(path, fp)
        # rewrite the file up to its last complete row (drops a torn tail)
        with open(path) as f:
            keep = f.read().split("\n")[: 2 + done]
        with open(path, "w") as f:
            f.write("\n".join(keep) + "\n")
    else:
        done, acc = 0, np.zeros(len(ROWS), dtype=np.uint64)
        with open(path, "w") as f:
            f.write(fp + "\n" + HEADER + "\n")
    n_chunks = 0
    with open(path, "a") as f:
        while done < len(xs):
            if max_chunks is not None and n_chunks >= max_chunks:
                break
            start = int(xs[done - 1]) if done else lo
            part = xs[done: done + chunk]
            res = count_fn(start, part)
            lines = []
            for i, x in enumerate(part):
                vals = acc + np.array([int(res[r][i]) for r in ROWS], dtype=np.uint64)
                lines.append(f"{int(x)}," + ",".join(str(int(v)) for v in vals))
            acc = acc + np.array([int(res[r][-1]) for r in ROWS], dtype=np.uint64)
            f.write("\n".join(lines) + "\n")
            f.flush()
            os.fsync(f.fileno())
            done += len(part)
            n_chunks += 1
    return done
