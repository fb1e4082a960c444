"""The paper's Algorithm 3 on the GPU: the chunked signature hash table.

Device counterpart of the reference's ``SignatureTable`` (chunked.py:129-304,
_kernels.py:130-232) and of its per-chunk search (chunked.py:307-359): open addressing with
the reference's slot word ((t+1) << 32 | home, 0 = empty), its commutative hash and linear
probing, but built by all GPU threads at once with 64-bit CAS.  The pair set equals the
serial build's and slot placement can differ; the pairs come back in the serial build's
discovery order all the same, restored by sorting: the serial build meets the stored entries
of one signature in insertion order along their probe chain, so its matches are ordered by
(n, m), and a serial probe's by (m, n) (the reference's golden lists, checked in order by
tests/test_gpu_table.py).

This path exists for an apples-to-apples comparison with the paper's method (it is
quadratic in the limit, like the reference); the production search is ``search.py``.
"""
from __future__ import annotations

import ctypes
import math
from typing import Callable, Iterator

import numpy as np

from . import _native
from .chunked import TableFullError, chunk_bounds, num_chunks, table_size_for
from .signatures import BeneluxPair, pairs_from_rows

_u64p = ctypes.POINTER(ctypes.c_uint64)


def _check(status: int) -> int:
    if status == _native.BNX_TABLE_FULL:
        raise TableFullError(_native.last_error())
    return _native.check(status)


class SignatureTable:
    """Device-resident signature table of one domain (API of chunked.py:129-304)."""

    def __init__(self, domain_start: int, rad_of: np.ndarray, rad_next: np.ndarray, *,
                 table_size: int | None = None, device: int | None = None):
        if len(rad_of) != len(rad_next):
            raise ValueError("radical arrays must have equal length")
        if len(rad_of) > 2**32 - 2:
            raise ValueError("domain too large for 32-bit slot offsets")
        if table_size is None:
            table_size = table_size_for(max(1, len(rad_of)))
        if table_size & (table_size - 1):
            raise ValueError("table size must be a power of two")
        if table_size > 2**32:
            raise ValueError("table too large for 32-bit home slots")
        self.ctx = _native.context(device)
        handle = ctypes.c_void_p()
        _check(_native.load().bnx_table_create(self.ctx.handle, table_size, ctypes.byref(handle)))
        self.handle = handle
        self.mask = table_size - 1
        self.domain_start = domain_start
        self.rad_of = np.ascontiguousarray(rad_of, np.uint64)
        self.rad_next = np.ascontiguousarray(rad_next, np.uint64)
        self.occupied = 0

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _native.load().bnx_table_destroy(self.handle)
        except Exception:
            pass

    @property
    def table_size(self) -> int:
        return self.mask + 1

    @property
    def load_factor(self) -> float:
        return self.occupied / self.table_size

    @property
    def slots(self) -> np.ndarray:
        out = np.empty(self.table_size, np.uint64)
        _check(_native.load().bnx_table_slots(self.handle, out.ctypes.data_as(_u64p), out.size))
        return out

    def reset_for_domain(self, domain_start: int, rad_of: np.ndarray, rad_next: np.ndarray) -> None:
        if len(rad_of) != len(rad_next) or len(rad_of) > 2**32 - 2:
            raise ValueError("bad radical arrays")
        if 4 * len(rad_of) > self.table_size:
            raise ValueError("table too small for this domain")
        self.domain_start = domain_start
        self.rad_of = np.ascontiguousarray(rad_of, np.uint64)
        self.rad_next = np.ascontiguousarray(rad_next, np.uint64)
        self.occupied = 0

    def _rows(self, fn) -> np.ndarray:
        cap = 256
        while True:
            buf = (_native.PairRow * cap)()
            found = ctypes.c_size_t(0)
            with self.ctx.lock:
                st = _check(fn(buf, cap, ctypes.byref(found)))
            if st == _native.BNX_BUFFER_FULL:
                cap = int(found.value)
                continue
            return np.frombuffer(buf, dtype=_native.PAIR_DTYPE, count=int(found.value)).copy()

    def insert_all(self, *, n_limit: int | None = None) -> list[BeneluxPair]:
        """Insert the whole domain (n < n_limit); every equal-signature pair, sorted by (n, m)."""
        limit = 2**64 - 1 if n_limit is None else n_limit
        inserted = ctypes.c_uint64(0)
        rows = self._rows(lambda b, c, f: _native.load().bnx_table_insert_all(
            self.handle, self.domain_start, self.rad_of.ctypes.data_as(_u64p), self.rad_next.ctypes.data_as(_u64p),
            self.rad_of.size, limit, b, c, f, ctypes.byref(inserted)))
        self.occupied = int(inserted.value)
        return pairs_from_rows(rows)

    def probe_all(self, probe_start: int, rad_of: np.ndarray, rad_next: np.ndarray) -> list[BeneluxPair]:
        """Pairs (m, n) for every probing m sharing a stored signature, sorted by (m, n)."""
        ro = np.ascontiguousarray(rad_of, np.uint64)
        rn = np.ascontiguousarray(rad_next, np.uint64)
        rows = self._rows(lambda b, c, f: _native.load().bnx_table_probe_all(
            self.handle, probe_start, ro.ctypes.data_as(_u64p), rn.ctypes.data_as(_u64p), ro.size, b, c, f))
        return pairs_from_rows(rows)


def search_chunk_table(index: int, chunk_size: int, *, n_limit: int | None = None, j_lo: int = 0,
                       j_hi: int | None = None, device: int | None = None) -> list[BeneluxPair]:
    """chunked.py:307-359 with Algorithm 3 on the device (sorted by (n, m))."""
    if chunk_size < 3:
        raise ValueError("chunk size must be >= 3")
    if chunk_size - 1 > 1 << 30:  # table_size_for would exceed 2^32 slots (chunked.py:157-158)
        raise ValueError("chunk size too large for 32-bit table slots")
    ctx = _native.context(device)
    hi = index if j_hi is None else j_hi
    limit = 2**64 - 1 if n_limit is None else n_limit
    cap = 256
    while True:
        buf = (_native.PairRow * cap)()
        found = ctypes.c_size_t(0)
        with ctx.lock:
            st = _check(_native.load().bnx_table_search_chunk(ctx.handle, index, chunk_size, limit, j_lo, hi, buf,
                                                               cap, ctypes.byref(found)))
        if st == _native.BNX_BUFFER_FULL:
            cap = int(found.value)
            continue
        return pairs_from_rows(np.frombuffer(buf, dtype=_native.PAIR_DTYPE, count=int(found.value)))


def run_full_chunked_table(limit: int, chunk_size: int, *, resume_from: int = 0,
                           on_chunk_done: Callable[[int], None] | None = None,
                           device: int | None = None) -> Iterator[BeneluxPair]:
    """chunked.py:362-412 with Algorithm 3 on the device: quadratic in limit / chunk_size."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    if chunk_size < 3:
        raise ValueError("chunk size must be >= 3")
    for index in range(resume_from, num_chunks(limit, chunk_size)):
        yield from search_chunk_table(index, chunk_size, n_limit=limit, device=device)
        if on_chunk_done is not None:
            on_chunk_done(index)
