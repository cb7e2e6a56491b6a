"""ctypes wrapper for oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Loads the C oracle (oracle/eis_oracle.c, see its header for the citations).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may use it.  No CUDA, no product code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "eis_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

NOT_IN_D = 0xFF


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, OpenMP). Building the checker is not using it."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", SRC, "-o", tmp]
        )
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        u64, i64, c_int = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
        vp = ctypes.c_void_p
        L.eo_is_squarefree.argtypes = [u64]
        L.eo_is_squarefree.restype = c_int
        L.eo_residue.argtypes = [u64, ctypes.POINTER(i64)]
        L.eo_residue.restype = c_int
        L.eo_unit.argtypes = [u64, vp, ctypes.POINTER(c_int), vp, ctypes.POINTER(c_int), c_int,
                              ctypes.POINTER(c_int), ctypes.POINTER(i64)]
        L.eo_unit.restype = c_int
        L.eo_classify_range.argtypes = [u64, u64, vp, i64, c_int]
        L.eo_classify_range.restype = i64
        L.eo_classify_list.argtypes = [vp, i64, vp, c_int]
        L.eo_classify_list.restype = c_int
        L.eo_count_window.argtypes = [u64, vp, i64, vp, vp, c_int]
        L.eo_count_window.restype = c_int
        _lib = L
    return _lib


def is_squarefree(d: int) -> bool:
    return bool(lib().eo_is_squarefree(d))


def residue(d: int) -> int:
    per = ctypes.c_int64()
    t = lib().eo_residue(d, ctypes.byref(per))
    if t < 0:
        raise ValueError(f"oracle error {t} for d={d}")
    return t


def fundamental_unit(d: int, cap: int = 1 << 16) -> tuple[int, int, int, int]:
    """(x0, y0, norm_sign, period) as Python ints."""
    x = np.zeros(cap, dtype=np.uint64)
    y = np.zeros(cap, dtype=np.uint64)
    nx, ny, norm = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    per = ctypes.c_int64()
    rc = lib().eo_unit(d, x.ctypes.data, ctypes.byref(nx), y.ctypes.data, ctypes.byref(ny), cap,
                       ctypes.byref(norm), ctypes.byref(per))
    if rc != 0:
        raise ValueError(f"oracle error {rc} for d={d}")

    def to_int(a, n):
        return sum(int(a[i]) << (64 * i) for i in range(n))

    return to_int(x, nx.value), to_int(y, ny.value), norm.value, per.value


def classify_range(lo: int, hi: int, nthreads: int = 0) -> np.ndarray:
    first = lo + ((5 - lo) % 8)
    n = 0 if first > hi else (hi - first) // 8 + 1
    out = np.empty(max(n, 1), dtype=np.uint8)
    r = lib().eo_classify_range(lo, hi, out.ctypes.data, n, nthreads)
    if r < 0:
        raise ValueError(f"oracle error {r}")
    return out[:n]


def classify_list(ds, nthreads: int = 0) -> np.ndarray:
    d = np.ascontiguousarray(np.asarray(ds, dtype=np.uint64))
    out = np.empty(max(len(d), 1), dtype=np.uint8)
    rc = lib().eo_classify_list(d.ctypes.data, len(d), out.ctypes.data, nthreads)
    if rc < 0:
        raise ValueError(f"oracle error {rc}")
    return out[: len(d)]


def count_window(lo: int, xs, nthreads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    x = np.ascontiguousarray(np.asarray(xs, dtype=np.uint64))
    cD = np.zeros(len(x), dtype=np.uint64)
    cE = np.zeros(len(x), dtype=np.uint64)
    rc = lib().eo_count_window(lo, x.ctypes.data, len(x), cD.ctypes.data, cE.ctypes.data,
                               nthreads)
    if rc < 0:
        raise ValueError(f"oracle error {rc}")
    return cD, cE
