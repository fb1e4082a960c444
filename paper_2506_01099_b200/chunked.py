"""Chunk-by-chunk streaming search -- drop-in for the reference's ``chunked.py``.

Keeps the reference's chunk geometry (Chunk :42-67, chunk_bounds :70-78, num_chunks :81-83,
table_size_for :86-90), hash (commutative_hash :93-101), per-chunk contract
(search_chunk :307-359: exactly the pairs whose n lies in the chunk's domain, sorted by
(n, m)) and streaming contract (run_full_chunked :362-412: chunks in order, on_chunk_done
after each chunk's pairs).  The B200 engine finds a domain's pairs without re-sieving
earlier chunks (their partners lie on residue classes verified exactly), so the run is
linear in the limit instead of quadratic; consecutive chunks are batched into one device
search of at least BATCH_INTEGERS integers.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Iterator

from .primes import PrimeList
from .search import search_rows
from .signatures import BeneluxPair, PairSignature, pairs_from_rows

DEFAULT_CHUNK_SIZE = 1 << 27

_MASK64 = (1 << 64) - 1
HASH_CONSTANTS = (0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB)

# Integers one device search covers at minimum when streaming many small chunks.
BATCH_INTEGERS = 1 << 32


class TableFullError(RuntimeError):
    """A probe wrapped the whole table (kept for API compatibility)."""


@dataclass(frozen=True)
class Chunk:
    """Interval [first, last]; consecutive chunks overlap in one integer and the domains
    [first, last-1] tile [1, inf)."""

    index: int
    size: int
    first: int
    last: int

    @property
    def domain_first(self) -> int:
        return self.first

    @property
    def domain_last(self) -> int:
        return self.last - 1

    @property
    def domain_count(self) -> int:
        return self.size - 1


def chunk_bounds(index: int, chunk_size: int) -> Chunk:
    if chunk_size < 3:
        raise ValueError("chunk size must be >= 3")
    if index < 0:
        raise ValueError("chunk index must be >= 0")
    first = 1 + index * (chunk_size - 1)
    last = 1 + (index + 1) * (chunk_size - 1)
    return Chunk(index=index, size=chunk_size, first=first, last=last)


def num_chunks(limit: int, chunk_size: int) -> int:
    """Chunks needed so the set-domains cover 1 .. limit-1."""
    return (limit - 2) // (chunk_size - 1) + 1


def table_size_for(domain_count: int) -> int:
    """Smallest power of two >= 4 * domain_count (load factor <= 1/4)."""
    if domain_count < 1:
        raise ValueError("domain must hold at least one element")
    return 1 << (4 * domain_count - 1).bit_length()


def _slot_of(lo: int, hi: int, mask: int, constants: tuple[int, int, int]) -> int:
    phi, mul1, mul2 = constants
    x = lo ^ (hi * phi & _MASK64)
    x = (x ^ (x >> 30)) * mul1 & _MASK64
    x = (x ^ (x >> 27)) * mul2 & _MASK64
    return (x ^ (x >> 31)) & mask


def commutative_hash(sig: PairSignature, table_size: int) -> int:
    """Slot index in [0, table_size) of a canonical signature; table_size a power of two."""
    if table_size & (table_size - 1) or table_size < 1:
        raise ValueError("table size must be a power of two")
    return _slot_of(sig.lo, sig.hi, table_size - 1, HASH_CONSTANTS)


def _domain(chunk: Chunk, n_limit: int | None) -> tuple[int, int] | None:
    lo, hi = chunk.domain_first, chunk.domain_last
    if n_limit is not None:
        hi = min(hi, n_limit - 1)
    return (lo, hi) if hi >= lo else None


def search_chunk(
    index: int,
    chunk_size: int,
    primes: PrimeList | None = None,
    *,
    n_limit: int | None = None,
    threads: int = 1,
    executor=None,
    table=None,
    device: int | None = None,
) -> list[BeneluxPair]:
    """All pairs (m, n), m < n, whose n lies in this chunk's set-domain, sorted by (n, m).

    ``threads``, ``executor`` and ``table`` are accepted for signature compatibility; the
    device does the work."""
    chunk = chunk_bounds(index, chunk_size)
    need = math.isqrt(chunk.last)
    if primes is not None and not primes.covers(need):
        raise ValueError(f"prime list covers {primes.limit} but interval endpoint needs {need}")
    dom = _domain(chunk, n_limit)
    if dom is None:
        return []
    return pairs_from_rows(search_rows(dom[0], dom[1], primes=primes, device=device))


def _prepare_run(limit: int, primes: PrimeList | None, device: int | None) -> None:
    """Build the device tables once for the run's final bound; the batch searches (rising
    bounds) then reuse them instead of rebuilding per batch."""
    from . import _native

    _native.context(device).prepare(limit, None if primes is None else primes.primes,
                                    0 if primes is None else primes.limit)


def run_full_chunked(
    limit: int,
    chunk_size: int = DEFAULT_CHUNK_SIZE,
    primes: PrimeList | None = None,
    *,
    resume_from: int = 0,
    threads: int = 1,
    on_chunk_done: Callable[[int], None] | None = None,
    device: int | None = None,
) -> Iterator[BeneluxPair]:
    """Stream every pair with m < n < limit, chunk by chunk (each chunk sorted by (n, m));
    on_chunk_done(i) fires after chunk i's pairs have all been yielded."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    if chunk_size < 3:
        raise ValueError("chunk size must be >= 3")
    total = num_chunks(limit, chunk_size)
    if primes is not None:
        need = math.isqrt(chunk_bounds(total - 1, chunk_size).last)
        if not primes.covers(need):
            raise ValueError(f"prime list covers {primes.limit} but interval endpoint needs {need}")
    per_batch = max(1, BATCH_INTEGERS // (chunk_size - 1))
    if resume_from < total:
        _prepare_run(limit, primes, device)
    index = resume_from
    while index < total:
        stop = min(total, index + per_batch)
        lo = chunk_bounds(index, chunk_size).domain_first
        hi = min(chunk_bounds(stop - 1, chunk_size).domain_last, limit - 1)
        rows = search_rows(lo, hi, primes=primes, device=device) if hi >= lo else []
        pos = 0
        for i in range(index, stop):
            dom_last = chunk_bounds(i, chunk_size).domain_last
            end = pos
            while end < len(rows) and int(rows[end]["n"]) <= dom_last:
                end += 1
            yield from pairs_from_rows(rows[pos:end])
            pos = end
            if on_chunk_done is not None:
                on_chunk_done(i)
        index = stop
