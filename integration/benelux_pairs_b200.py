"""B200 backend for the reference package -- the file a `benelux_pairs` maintainer adds.

Drop it into the reference as ``benelux_pairs/_b200.py``.  It
binds ``libbenelux_b200.so`` (include/benelux_b200.h) with ctypes and returns the REFERENCE's
own result types (``benelux_pairs.signatures.BeneluxPair`` / ``Kind``), so the front-ends can
dispatch to it without any other change:

    sort_search.find_pairs_sorted  (sort_search.py:37-91)   -> find_pairs_sorted
    chunked.search_chunk           (chunked.py:307-359)     -> search_chunk
    chunked.run_full_chunked       (chunked.py:362-412)     -> run_full_chunked
    radical.sieve_radicals         (radical.py:109-124)     -> sieve_values

It depends only on ctypes, numpy and the reference's ``signatures`` module -- not on the
``paper_2506_01099_b200`` package.  The library is found through $BNX_LIB, else next to this
repo's package.  Errors follow the reference: ValueError for bad arguments or a prime list
that does not cover the interval (radical.py:119-120), RuntimeError for device failures.
Executed by tests/test_integration.py (CPU: binding) and tests/test_gpu_integration.py
(GPU: the reference's golden rows through this module).
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

try:  # inside the reference package (benelux_pairs/_b200.py)
    from .signatures import BeneluxPair, Kind  # type: ignore[import-not-found]
except ImportError:  # standalone: the reference importable as `benelux_pairs`
    from benelux_pairs.signatures import BeneluxPair, Kind  # type: ignore[no-redef]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BNX_LIB") or os.path.join(os.path.dirname(_HERE), "paper_2506_01099_b200",
                                                      "libbenelux_b200.so")

BNX_OK, BNX_TABLE_FULL, BNX_BUFFER_FULL = 0, 1, 2
BNX_ERR_PRIMES_UNCOVERED, BNX_ERR_INVALID, BNX_ERR_CUDA, BNX_ERR_RANGE = 3, 4, 5, 6
BOTH_KINDS = 3  # the reference always reports both kinds


class _Pair(ctypes.Structure):  # bnx_pair_t
    _fields_ = [("m", ctypes.c_uint64), ("n", ctypes.c_uint64), ("rad_m", ctypes.c_uint64),
                ("rad_m1", ctypes.c_uint64), ("kind", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_u64p = ctypes.POINTER(ctypes.c_uint64)
_szp = ctypes.POINTER(ctypes.c_size_t)
_vp = ctypes.c_void_p
_lock = threading.Lock()
_lib = None
_ctx = None

# the entry points this module calls, with their ctypes signatures
SIGNATURES = {
    "bnx_last_error": ([], ctypes.c_char_p),
    "bnx_ctx_create": ([ctypes.c_int, ctypes.POINTER(_vp)], ctypes.c_int),
    "bnx_search": ([_vp, ctypes.c_uint64, ctypes.c_uint32, _u64p, ctypes.c_size_t, ctypes.c_uint64,
                    ctypes.POINTER(_Pair), ctypes.c_size_t, _szp], ctypes.c_int),
    "bnx_search_domain": ([_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, _u64p, ctypes.c_size_t,
                           ctypes.c_uint64, ctypes.POINTER(_Pair), ctypes.c_size_t, _szp], ctypes.c_int),
    "bnx_sieve_radicals": ([_vp, ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_uint64,
                            ctypes.c_int, _u64p], ctypes.c_int),
}


def library() -> ctypes.CDLL:
    """The bound library (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes, fn.restype = args, res
            _lib = lib
    return _lib


def _context():
    global _ctx
    lib = library()
    with _lock:
        if _ctx is None:
            h = _vp()
            _check(lib.bnx_ctx_create(int(os.environ.get("BNX_DEVICE", "0")), ctypes.byref(h)))
            _ctx = h
    return _ctx


def _check(status: int) -> int:
    if status in (BNX_OK, BNX_BUFFER_FULL):
        return status
    msg = (library().bnx_last_error() or b"").decode()
    if status in (BNX_ERR_PRIMES_UNCOVERED, BNX_ERR_INVALID, BNX_ERR_RANGE):
        raise ValueError(msg)
    raise RuntimeError(msg or f"libbenelux_b200 status {status}")


def _pairs(call) -> list:
    """Rows -> the reference's BeneluxPair, with the reference's capacity x4 retry on
    BUFFER_FULL (chunked.py:268-270)."""
    cap = 256
    while True:
        buf, found = (_Pair * cap)(), ctypes.c_size_t(0)
        if _check(call(buf, cap, ctypes.byref(found))) == BNX_BUFFER_FULL:
            cap = max(4 * cap, int(found.value))
            continue
        return [BeneluxPair(r.m, r.n, Kind(r.kind), r.rad_m, r.rad_m1) for r in buf[: found.value]]


def _prime_args(primes):
    """(keep-alive array, pointer, count, PrimeList.limit) of an optional reference PrimeList."""
    if primes is None:
        return None, None, 0, 0
    arr = np.ascontiguousarray(primes.primes, dtype=np.uint64)
    return arr, arr.ctypes.data_as(_u64p), int(arr.size), int(primes.limit)


def find_pairs_sorted(limit: int, primes=None) -> list:
    """sort_search.find_pairs_sorted (sort_search.py:37-91): every pair m < n < limit, both
    kinds, sorted by (m, n).  `primes` (a PrimeList) must cover isqrt(limit) when given."""
    keep, pp, npr, plim = _prime_args(primes)  # noqa: F841
    ctx = _context()
    return _pairs(lambda b, c, f: library().bnx_search(ctx, limit, BOTH_KINDS, pp, npr, plim, b, c, f))


def _chunk_domain(index: int, chunk_size: int) -> tuple[int, int]:
    """Set-domain [first, last - 1] of chunk C_i = [1 + i (s - 1), 1 + (i + 1)(s - 1)]
    (chunked.py:42-78)."""
    first = 1 + index * (chunk_size - 1)
    return first, first + chunk_size - 2


def search_chunk(index: int, chunk_size: int, primes=None, *, n_limit: int | None = None, threads: int = 1,
                 executor=None, table=None) -> list:
    """chunked.search_chunk (chunked.py:307-359): every pair (m, n), m < n, with n in chunk
    `index`'s domain (and n < n_limit), sorted by (n, m).  The device needs no table and no
    earlier chunks, so `threads`, `executor` and `table` have nothing to do."""
    if chunk_size < 3 or index < 0:
        raise ValueError("chunk size must be >= 3 and index >= 0")
    lo, hi = _chunk_domain(index, chunk_size)
    if n_limit is not None:
        hi = min(hi, n_limit - 1)
    if hi < lo:
        return []
    keep, pp, npr, plim = _prime_args(primes)  # noqa: F841
    ctx = _context()
    return _pairs(lambda b, c, f: library().bnx_search_domain(ctx, lo, hi, BOTH_KINDS, pp, npr, plim, b, c, f))


def run_full_chunked(limit: int, chunk_size: int = 2**27, primes=None, *, resume_from: int = 0, threads: int = 1,
                     on_chunk_done=None):
    """chunked.run_full_chunked (chunked.py:362-412): the pairs with m < n < limit chunk by
    chunk (each chunk sorted by (n, m)), calling on_chunk_done(i) after chunk i's pairs."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    if chunk_size < 3:
        raise ValueError("chunk size must be >= 3")
    total = (limit - 2) // (chunk_size - 1) + 1  # num_chunks (chunked.py:81-83)
    for index in range(resume_from, total):
        yield from search_chunk(index, chunk_size, primes, n_limit=limit)
        if on_chunk_done is not None:
            on_chunk_done(index)


def sieve_values(start: int, length: int, primes, ctz_fast_path: bool = True) -> np.ndarray:
    """radical.sieve_radicals' kernel call (radical.py:109-124, _kernels.sieve_segment
    _kernels.py:48-84): rad(start + k) for k < length as uint64.  `primes` is the caller's
    PrimeList; its real `limit` is passed, so a list that does not cover isqrt(start + length
    - 1) is refused by the library (ValueError), exactly as radical.py:119-120 refuses it."""
    if start < 1 or length < 1:
        raise ValueError("interval must start at 1 or above and be non-empty")
    keep, pp, npr, plim = _prime_args(primes)  # noqa: F841
    if keep is None:
        raise ValueError("sieve_values needs the caller's PrimeList")
    out = np.empty(length, np.uint64)
    _check(library().bnx_sieve_radicals(_context(), start, length, pp, npr, plim, int(bool(ctz_fast_path)),
                                        out.ctypes.data_as(_u64p)))
    return out


def required_prime_bound(start: int, length: int) -> int:
    """radical.required_prime_bound (radical.py:104-106) for [start, start + length)."""
    return math.isqrt(start + length - 1)
