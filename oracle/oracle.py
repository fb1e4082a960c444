"""ctypes front end of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg, never by the product package
``paper_2506_01099_b200``.  Each wrapper names the reference function it restates;
the C source cites the reference file:line.  The restatement is pinned against the
reference's own golden vectors by tests/test_oracle_golden.py.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import NamedTuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

STATUS_OK, STATUS_TABLE_FULL, STATUS_BUFFER_FULL, STATUS_NOMEM = 0, 1, 2, 3
HASH_CONSTANTS = (0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB)

_u64p = ctypes.POINTER(ctypes.c_uint64)


class _Pairs(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.POINTER(ctypes.c_int8)),
        ("m", _u64p),
        ("n", _u64p),
        ("rm", _u64p),
        ("rm1", _u64p),
        ("cap", ctypes.c_size_t),
        ("found", ctypes.c_size_t),
    ]


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
            os.path.join(HERE, "oracle.c")
        ):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_primes_up_to.restype = ctypes.c_int64
        L.orc_primes_up_to.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t]
        L.orc_sieve_segment.argtypes = [ctypes.c_uint64, ctypes.c_size_t, _u64p, ctypes.c_size_t, ctypes.c_int, _u64p]
        L.orc_radicals_trial_division.argtypes = [ctypes.c_uint64, ctypes.c_size_t, _u64p]
        L.orc_strip_twos.argtypes = [_u64p, ctypes.c_size_t, ctypes.c_uint64]
        L.orc_slot_of.restype = ctypes.c_uint64
        L.orc_slot_of.argtypes = [ctypes.c_uint64] * 6
        L.orc_build_table.restype = ctypes.c_int
        L.orc_build_table.argtypes = [
            ctypes.c_uint64, _u64p, _u64p, ctypes.c_size_t, ctypes.c_uint64, _u64p,
            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
            ctypes.POINTER(_Pairs), ctypes.POINTER(ctypes.c_size_t),
        ]
        L.orc_probe_table.restype = ctypes.c_int
        L.orc_probe_table.argtypes = [
            ctypes.c_uint64, _u64p, _u64p, ctypes.c_size_t, ctypes.c_uint64, _u64p, _u64p, _u64p,
            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(_Pairs),
        ]
        L.orc_brute_force_scan.restype = ctypes.c_int
        L.orc_brute_force_scan.argtypes = [_u64p, ctypes.c_size_t, ctypes.POINTER(_Pairs)]
        L.orc_find_pairs_sorted.restype = ctypes.c_int
        L.orc_find_pairs_sorted.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.POINTER(_Pairs)]
        L.orc_search_chunk.restype = ctypes.c_int
        L.orc_search_chunk.argtypes = [
            ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int,
            ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_uint64, _u64p, ctypes.POINTER(_Pairs),
            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
        ]
        L.orc_build_chunk.restype = ctypes.c_int
        L.orc_build_chunk.argtypes = [
            ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_uint64, _u64p, ctypes.c_uint64,
            _u64p, ctypes.POINTER(_Pairs), ctypes.POINTER(ctypes.c_double),
        ]
        L.orc_probe_chunks.restype = ctypes.c_int
        L.orc_probe_chunks.argtypes = [
            ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64,
            ctypes.c_uint64, _u64p, ctypes.c_uint64, _u64p, ctypes.c_uint64, ctypes.POINTER(_Pairs),
            ctypes.POINTER(ctypes.c_double),
        ]
        L.orc_run_full_chunked.restype = ctypes.c_int
        L.orc_run_full_chunked.argtypes = [
            ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int,
            ctypes.POINTER(_Pairs), _u64p,
        ]
        L.orc_num_chunks.restype = ctypes.c_uint64
        L.orc_num_chunks.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.orc_table_size_for.restype = ctypes.c_uint64
        L.orc_table_size_for.argtypes = [ctypes.c_uint64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_u64p)


class PairBuffers:
    """The five caller-allocated match buffers of chunked.py:112-119."""

    def __init__(self, capacity: int):
        self.kind = np.zeros(capacity + 1, np.int8)
        self.m = np.zeros(capacity + 1, np.uint64)
        self.n = np.zeros(capacity + 1, np.uint64)
        self.rm = np.zeros(capacity + 1, np.uint64)
        self.rm1 = np.zeros(capacity + 1, np.uint64)
        self.s = _Pairs(
            self.kind.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
            _p(self.m), _p(self.n), _p(self.rm), _p(self.rm1), capacity, 0,
        )

    def rows(self) -> list[tuple[int, int, int, int, int]]:
        k = min(self.s.found, self.s.cap)
        return [
            (int(self.kind[t]), int(self.m[t]), int(self.n[t]), int(self.rm[t]), int(self.rm1[t]))
            for t in range(k)
        ]


def _with_retry(fn, capacity: int = 256):
    """BUFFER_FULL -> capacity x4 and re-run from scratch (chunked.py:249-270)."""
    while True:
        buf = PairBuffers(capacity)
        status = fn(buf)
        if status == STATUS_BUFFER_FULL:
            capacity *= 4
            continue
        if status == STATUS_TABLE_FULL:
            raise RuntimeError("table full")
        if status == STATUS_NOMEM:
            raise MemoryError("oracle out of memory")
        return buf.rows()


# ---------------------------------------------------------------------------------------
def primes_up_to(limit: int) -> np.ndarray:
    """primes.py:24-35."""
    if limit < 2:
        return np.empty(0, np.uint64)
    cap = int(1.3 * limit / max(1.0, math.log(limit))) + 64
    out = np.empty(cap, np.uint64)
    count = lib().orc_primes_up_to(limit, _p(out), cap)
    return out[:count].copy()


def sieve_segment(start: int, length: int, primes: np.ndarray, fast_two: bool = True) -> np.ndarray:
    """_kernels.sieve_segment (_kernels.py:48-84)."""
    primes = np.ascontiguousarray(primes, np.uint64)
    out = np.empty(length, np.uint64)
    lib().orc_sieve_segment(start, length, _p(primes), primes.size, int(fast_two), _p(out))
    return out


def strip_twos(vals: np.ndarray, start: int) -> np.ndarray:
    """_kernels.strip_twos (_kernels.py:33-45), in place; returns vals."""
    lib().orc_strip_twos(_p(vals), vals.size, start)
    return vals


def radicals_trial_division(start: int, length: int) -> np.ndarray:
    """_kernels.radicals_trial_division (_kernels.py:87-112)."""
    out = np.empty(length, np.uint64)
    lib().orc_radicals_trial_division(start, length, _p(out))
    return out


def slot_of(lo: int, hi: int, mask: int, constants=HASH_CONSTANTS) -> int:
    """_kernels._slot_of (_kernels.py:115-123)."""
    return int(lib().orc_slot_of(lo, hi, mask, *constants))


def brute_force(limit: int) -> list[tuple[int, int, int, int, int]]:
    """bruteforce.brute_force_pairs (bruteforce.py:16-42) -> rows sorted by (m, n)."""
    rads = radicals_trial_division(1, limit)
    rows = _with_retry(lambda b: lib().orc_brute_force_scan(_p(rads), limit, ctypes.byref(b.s)))
    return sorted(rows, key=lambda r: (r[1], r[2]))


def find_pairs_sorted(limit: int) -> list[tuple[int, int, int, int, int]]:
    """sort_search.find_pairs_sorted (sort_search.py:37-91) -> rows sorted by (m, n)."""
    primes = primes_up_to(math.isqrt(limit))
    rows = _with_retry(lambda b: lib().orc_find_pairs_sorted(limit, _p(primes), primes.size, ctypes.byref(b.s)))
    return sorted(rows, key=lambda r: (r[1], r[2]))


def run_full_chunked(limit: int, chunk_size: int, *, threads: int = 1, resume_from: int = 0):
    """chunked.run_full_chunked (chunked.py:362-412) -> rows, chunk by chunk, each chunk
    sorted by (n, m) (chunked.py:358)."""
    if limit < 3 or chunk_size < 3:
        raise ValueError("limit and chunk size must be >= 3")
    total = int(lib().orc_num_chunks(limit, chunk_size))
    last = 1 + total * (chunk_size - 1)
    primes = primes_up_to(math.isqrt(last))
    capacity = 256
    while True:
        buf = PairBuffers(capacity)
        ends = np.zeros(max(1, total - resume_from), np.uint64)
        st = lib().orc_run_full_chunked(
            limit, chunk_size, _p(primes), primes.size, resume_from, threads, ctypes.byref(buf.s), _p(ends)
        )
        if st == STATUS_BUFFER_FULL:
            capacity *= 4
            continue
        if st != STATUS_OK:
            raise RuntimeError(f"oracle chunked run failed with status {st}")
        break
    rows = buf.rows()
    out, begin = [], 0
    for end in ends[: max(0, total - resume_from)].tolist():
        out.extend(sorted(rows[begin:int(end)], key=lambda r: (r[2], r[1])))
        begin = int(end)
    return out


def build_table(domain_start, rad_of, rad_next, n_limit, table_size, constants=HASH_CONSTANTS):
    """_kernels.build_table (_kernels.py:130-183) -> (rows, inserted, slots)."""
    rad_of = np.ascontiguousarray(rad_of, np.uint64)
    rad_next = np.ascontiguousarray(rad_next, np.uint64)
    capacity = 256
    while True:
        slots = np.zeros(table_size, np.uint64)
        buf = PairBuffers(capacity)
        inserted = ctypes.c_size_t(0)
        st = lib().orc_build_table(
            domain_start, _p(rad_of), _p(rad_next), rad_of.size, n_limit, _p(slots),
            table_size - 1, *constants, ctypes.byref(buf.s), ctypes.byref(inserted),
        )
        if st == STATUS_BUFFER_FULL:
            capacity *= 4
            continue
        if st == STATUS_TABLE_FULL:
            raise RuntimeError("table full")
        return buf.rows(), int(inserted.value), slots


def probe_table(probe_start, rad_of, rad_next, domain_start, cur_rad_of, cur_rad_next, slots,
                constants=HASH_CONSTANTS):
    """_kernels.probe_table (_kernels.py:186-232) -> rows."""
    arrs = [np.ascontiguousarray(a, np.uint64) for a in (rad_of, rad_next, cur_rad_of, cur_rad_next)]
    return _with_retry(
        lambda b: lib().orc_probe_table(
            probe_start, _p(arrs[0]), _p(arrs[1]), arrs[0].size, domain_start, _p(arrs[2]), _p(arrs[3]),
            _p(slots), slots.size - 1, *constants, ctypes.byref(b.s),
        )
    )


class ChunkSample(NamedTuple):
    t_build: float
    t_probe: float
    probes: int
    rows: list


def search_chunk_sample(index: int, chunk_size: int, limit: int, threads: int, j_lo: int, j_hi: int,
                        primes: np.ndarray, slots: np.ndarray, vals: np.ndarray) -> ChunkSample:
    """One chunked.search_chunk (chunked.py:307-359) restricted to earlier chunks j in
    [j_lo, j_hi): sieve + build of chunk `index`, then `j_hi-j_lo` re-sieve+probe tasks
    spread over `threads` pthreads.  Used by bench.py to time the reference on a bounded
    sample of a large run."""
    buf = PairBuffers(4096)
    tb, tp = ctypes.c_double(0), ctypes.c_double(0)
    st = lib().orc_search_chunk(
        index, chunk_size, _p(primes), primes.size, limit, threads, j_lo, j_hi, _p(slots), slots.size,
        _p(vals), ctypes.byref(buf.s), ctypes.byref(tb), ctypes.byref(tp),
    )
    if st not in (STATUS_OK, STATUS_BUFFER_FULL):
        raise RuntimeError(f"oracle search_chunk failed with status {st}")
    return ChunkSample(tb.value, tp.value, j_hi - j_lo, buf.rows())


class ChunkTable:
    """A built chunk table kept alive for repeated probe rounds (bench sampling):
    chunked.py:326-333 (build) then chunked.py:335-356 (probe) on demand."""

    def __init__(self, index: int, chunk_size: int, limit: int, primes: np.ndarray):
        self.index, self.s, self.primes = index, chunk_size, primes
        self.slots = np.zeros(table_size_for(chunk_size - 1), np.uint64)
        self.vals = np.zeros(chunk_size, np.uint64)
        buf = PairBuffers(4096)
        t = ctypes.c_double(0)
        st = lib().orc_build_chunk(index, chunk_size, _p(primes), primes.size, limit, _p(self.slots),
                                   self.slots.size, _p(self.vals), ctypes.byref(buf.s), ctypes.byref(t))
        if st not in (STATUS_OK, STATUS_BUFFER_FULL):
            raise RuntimeError(f"oracle build failed with status {st}")
        self.t_build = t.value
        self.build_rows = buf.rows()

    def probe(self, j_lo: int, j_hi: int, threads: int, sub_len: int = 0) -> tuple[float, list]:
        """Probe with earlier chunks j in [j_lo, j_hi); sub_len > 0 probes only the first
        sub_len values of each (a proportional sample of the same per-value work)."""
        buf = PairBuffers(4096)
        t = ctypes.c_double(0)
        st = lib().orc_probe_chunks(self.index, self.s, _p(self.primes), self.primes.size, threads, j_lo, j_hi,
                                    _p(self.slots), self.slots.size, _p(self.vals), sub_len, ctypes.byref(buf.s),
                                    ctypes.byref(t))
        if st not in (STATUS_OK, STATUS_BUFFER_FULL):
            raise RuntimeError(f"oracle probe failed with status {st}")
        return t.value, buf.rows()


def num_chunks(limit: int, chunk_size: int) -> int:
    return int(lib().orc_num_chunks(limit, chunk_size))


def table_size_for(count: int) -> int:
    return int(lib().orc_table_size_for(count))
