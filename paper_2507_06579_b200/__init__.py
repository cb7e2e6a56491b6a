"""B200-native Eisenstein-discriminant classifier (arXiv 2507.06579).

Thin Python binding over the C ABI in ``include/eis.h`` (``libeis.so``, built
in-tree for sm_100a).  Argument marshalling only: every step of the path --
sieve, compaction, residue walk, checkpoint histogram, prefix sums -- runs in
the library's CUDA kernels.  There is no CPU fallback: if the library is
missing or no device is usable, every call raises ``EisError``.

Names follow the ABI: ``classify_range``, ``count``, ``count_window``,
``count_buckets_dev``, ``prefix_dev``, ``classify_range_dev``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "EisError", "load", "init", "finalize", "set_option", "get_option", "num_candidates",
    "classify_range", "count", "count_window", "count_window_ext", "count_buckets_dev",
    "prefix_dev",
    "classify_range_dev", "get_stats", "MODE_AUTO", "MODE_HALF", "MODE_BSGS", "NOT_IN_D",
    "MAX_D", "LIB_PATH", "shard_bounds", "comm_unique_id", "comm_init", "comm_finalize",
    "count_window_comm", "BALANCE",
]

LIB_PATH = os.environ.get("EIS_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "libeis.so")   # EIS_LIB: build experiments
MAX_D = 100_000_000_000
NOT_IN_D = 0xFF
MODE_AUTO, MODE_HALF, MODE_BSGS = 0, 1, 2
BALANCE = {"flat": 0, "prefix": 1, "auto": 2}      # EIS_BALANCE_*
COMM_ID_BYTES = 128

EIS_OK, EIS_EINVAL, EIS_ERANGE, EIS_ENOMEM, EIS_EDEVICE, EIS_EINTERNAL = 0, -1, -2, -3, -4, -5
_CODES = {-1: "EINVAL", -2: "ERANGE", -3: "ENOMEM", -4: "EDEVICE", -5: "EINTERNAL"}

EXPORTS = (
    "eis_init", "eis_finalize", "eis_last_error", "eis_set_option", "eis_get_option",
    "eis_num_candidates", "eis_classify_range", "eis_count", "eis_count_window",
    "eis_count_buckets_dev", "eis_prefix_dev", "eis_classify_range_dev", "eis_get_stats",
    "eis_count_window_ext", "eis_shard_bounds", "eis_comm_unique_id", "eis_comm_init",
    "eis_comm_finalize", "eis_count_window_comm",
)
NROWS = 5
ROW_NAMES = ("D", "E", "T1", "DP", "EP")


class EisError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"eis {_CODES.get(code, code)}: {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [
        ("d_classified", ctypes.c_uint64),
        ("baby_steps", ctypes.c_uint64),
        ("giant_steps", ctypes.c_uint64),
        ("reduce_steps", ctypes.c_uint64),
        ("sym_exits", ctypes.c_uint64),
        ("fallbacks", ctypes.c_uint64),
        ("kernel_launches", ctypes.c_uint64),
        ("walk_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("sieve_ms", ctypes.c_double),
        ("window_ms", ctypes.c_double),
        ("giant_ms", ctypes.c_double),
        ("windowed", ctypes.c_uint64),
        ("window_nw", ctypes.c_uint64),
        ("window_nb", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load libeis.so (raises if it was not built: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EisError(EIS_EDEVICE, f"{LIB_PATH} not built; run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    u64, i64, c_int, vp, sz = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_size_t)
    L.eis_init.argtypes = [c_int]
    L.eis_init.restype = c_int
    L.eis_finalize.argtypes = []
    L.eis_finalize.restype = None
    L.eis_last_error.argtypes = []
    L.eis_last_error.restype = ctypes.c_char_p
    L.eis_set_option.argtypes = [ctypes.c_char_p, i64]
    L.eis_set_option.restype = c_int
    L.eis_get_option.argtypes = [ctypes.c_char_p]
    L.eis_get_option.restype = i64
    L.eis_num_candidates.argtypes = [u64, u64]
    L.eis_num_candidates.restype = sz
    L.eis_classify_range.argtypes = [u64, u64, vp, sz]
    L.eis_classify_range.restype = c_int
    L.eis_count.argtypes = [vp, sz, vp, vp]
    L.eis_count.restype = c_int
    L.eis_count_window.argtypes = [u64, vp, sz, vp, vp]
    L.eis_count_window.restype = c_int
    L.eis_count_window_ext.argtypes = [u64, vp, sz, vp]
    L.eis_count_window_ext.restype = c_int
    L.eis_count_buckets_dev.argtypes = [u64, u64, vp, sz, vp, vp]
    L.eis_count_buckets_dev.restype = c_int
    L.eis_prefix_dev.argtypes = [vp, sz, vp, vp]
    L.eis_prefix_dev.restype = c_int
    L.eis_classify_range_dev.argtypes = [u64, u64, vp, sz, vp]
    L.eis_classify_range_dev.restype = c_int
    L.eis_get_stats.argtypes = [ctypes.POINTER(Stats)]
    L.eis_get_stats.restype = c_int
    L.eis_shard_bounds.argtypes = [u64, u64, c_int, c_int, c_int, ctypes.POINTER(u64),
                                   ctypes.POINTER(u64)]
    L.eis_shard_bounds.restype = c_int
    L.eis_comm_unique_id.argtypes = [vp]
    L.eis_comm_unique_id.restype = c_int
    L.eis_comm_init.argtypes = [vp, c_int, c_int]
    L.eis_comm_init.restype = c_int
    L.eis_comm_finalize.argtypes = []
    L.eis_comm_finalize.restype = None
    L.eis_count_window_comm.argtypes = [u64, vp, sz, vp, vp]
    L.eis_count_window_comm.restype = c_int
    _lib = L
    return L


def _check(rc: int) -> int:
    if rc < 0:
        raise EisError(rc, load().eis_last_error().decode())
    return rc


def init(device: int = -1) -> None:
    _check(load().eis_init(device))


def finalize() -> None:
    load().eis_finalize()


def set_option(key: str, value: int) -> None:
    _check(load().eis_set_option(key.encode(), int(value)))


def get_option(key: str) -> int:
    return _check(load().eis_get_option(key.encode()))


def num_candidates(lo: int, hi: int) -> int:
    return load().eis_num_candidates(lo, hi)


def classify_range(lo: int, hi: int, out: np.ndarray | None = None) -> np.ndarray:
    """uint8 flags for d = first + 8i <= hi: t(eps_d) in {0,1,2} or NOT_IN_D."""
    n = num_candidates(lo, hi) if lo <= hi else 0
    if out is None:
        out = np.empty(n, dtype=np.uint8)
    _check(load().eis_classify_range(lo, hi, out.ctypes.data if n else None, out.size))
    return out[:n]


def _u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


def count(x) -> tuple[np.ndarray, np.ndarray]:
    """(pi_D(x_i), pi_E(x_i)) for ascending checkpoints x."""
    x = _u64(x)
    pD = np.zeros(len(x), dtype=np.uint64)
    pE = np.zeros(len(x), dtype=np.uint64)
    _check(load().eis_count(x.ctypes.data, len(x), pD.ctypes.data, pE.ctypes.data))
    return pD, pE


def count_window(lo: int, x) -> tuple[np.ndarray, np.ndarray]:
    """(#{d in D: lo < d <= x_i}, #{d in E: lo < d <= x_i})."""
    x = _u64(x)
    cD = np.zeros(len(x), dtype=np.uint64)
    cE = np.zeros(len(x), dtype=np.uint64)
    _check(load().eis_count_window(lo, x.ctypes.data, len(x), cD.ctypes.data, cE.ctypes.data))
    return cD, cE


def count_window_ext(lo: int, x) -> dict:
    """Rows D, E, T1 (t=1), DP (primes in D), EP (primes in E) over lo < d <= x_i
    (Sec. 3.2); T2 = D - E - T1."""
    x = _u64(x)
    out = np.zeros((NROWS, len(x)), dtype=np.uint64)
    _check(load().eis_count_window_ext(lo, x.ctypes.data, len(x), out.ctypes.data))
    return dict(zip(ROW_NAMES, out))


def _stream_handle(stream) -> int | None:
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream))


def count_buckets_dev(lo: int, hi: int, x, buckets, stream=None) -> None:
    """Accumulate bucket counts of d in (lo, hi] into ``buckets`` (a CUDA
    uint64/int64 tensor of 2*len(x) elements; not zeroed)."""
    x = _u64(x)
    assert buckets.is_cuda and buckets.numel() == 2 * len(x) and buckets.element_size() == 8
    _check(load().eis_count_buckets_dev(lo, hi, x.ctypes.data, len(x), buckets.data_ptr(),
                                        _stream_handle(stream)))


def prefix_dev(buckets, out, stream=None) -> None:
    n = buckets.numel() // 2
    _check(load().eis_prefix_dev(buckets.data_ptr(), n, out.data_ptr(), _stream_handle(stream)))


def classify_range_dev(lo: int, hi: int, out, stream=None) -> None:
    assert out.is_cuda and out.element_size() == 1
    _check(load().eis_classify_range_dev(lo, hi, out.data_ptr(), out.numel(),
                                         _stream_handle(stream)))


def get_stats() -> dict:
    s = Stats()
    _check(load().eis_get_stats(ctypes.byref(s)))
    return s.as_dict()


# ---- the whole box (include/eis.h "one process per GPU") ----
def shard_bounds(lo: int, hi: int, world: int, rank: int, balance: str = "flat") -> tuple[int, int]:
    """Contiguous shard (a, b] of (lo, hi] for ``rank`` of ``world`` (eis_shard_bounds;
    balance "flat", "prefix" or "auto").  Host-only."""
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    _check(load().eis_shard_bounds(lo, hi, world, rank, BALANCE[balance], ctypes.byref(a),
                                   ctypes.byref(b)))
    return int(a.value), int(b.value)


def comm_unique_id() -> bytes:
    """A new NCCL unique id (rank 0); broadcast it to the other ranks."""
    buf = ctypes.create_string_buffer(COMM_ID_BYTES)
    _check(load().eis_comm_unique_id(buf))
    return buf.raw


def comm_init(uid: bytes, world: int, rank: int) -> None:
    assert len(uid) == COMM_ID_BYTES
    buf = ctypes.create_string_buffer(uid, COMM_ID_BYTES)
    _check(load().eis_comm_init(buf, world, rank))


def comm_finalize() -> None:
    load().eis_comm_finalize()


def count_window_comm(lo: int, x) -> tuple[np.ndarray, np.ndarray]:
    """count_window over the library's NCCL communicator (collective)."""
    x = _u64(x)
    cD = np.zeros(len(x), dtype=np.uint64)
    cE = np.zeros(len(x), dtype=np.uint64)
    _check(load().eis_count_window_comm(lo, x.ctypes.data, len(x), cD.ctypes.data,
                                        cE.ctypes.data))
    return cD, cE
