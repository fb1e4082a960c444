"""Full search below a bound -- drop-in for the reference's ``sort_search.py``.

``find_pairs_sorted`` keeps the reference's signature and result (every pair m < n < limit,
both kinds, sorted by (m, n); sort_search.py:37-91) but runs the B200 search engine, which
needs no per-integer records: its device footprint is a few fixed buffers plus the prime
tables, so the memory budget check applies to that footprint.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from .primes import PrimeList
from .radical import RadicalSegment
from .search import find_pairs
from .signatures import BeneluxPair, PairSignature, signature_of

# Reference: values + lo + hi + sort order + two sorted key copies, all uint64 (sort_search.py:18).
# The device path keeps nothing per integer; kept for API compatibility.
BYTES_PER_RECORD = 48
DEFAULT_MEMORY_BUDGET = 14 * 2**30

# Fixed device work buffers of one search context (survivors, candidates, matches, pairs,
# counters) and bytes per prime-table entry (prime, progression, exact-division constants).
DEVICE_WORK_BYTES = (1 << 20) * 8 + (1 << 14) * 40 + 4096
DEVICE_BYTES_PER_PRIME = 4 + 24 + 24


class MemoryBudgetExceeded(ValueError):
    """The search would not fit the memory budget; use the chunked search."""


@dataclass(frozen=True)
class SignatureRecord:
    n: int
    sig: PairSignature


def signature_record(n: int, segment: RadicalSegment) -> SignatureRecord:
    """Record (n, signature of n) read off a radical segment."""
    return SignatureRecord(n, signature_of(n, segment.rad(n), segment.rad(n + 1)))


def device_bytes_for(limit: int) -> int:
    """Device memory one search below `limit` needs (work buffers + prime tables)."""
    root = math.isqrt(limit)
    primes_est = int(1.26 * root / max(1.0, math.log(max(root, 2)))) + 64
    return DEVICE_WORK_BYTES + DEVICE_BYTES_PER_PRIME * primes_est


def find_pairs_sorted(limit: int, primes: PrimeList | None = None, *,
                      memory_budget_bytes: int = DEFAULT_MEMORY_BUDGET, device: int | None = None
                      ) -> list[BeneluxPair]:
    """Every Benelux pair of either kind with m < n < limit, sorted by (m, n)."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    estimated = device_bytes_for(limit)
    if estimated > memory_budget_bytes:
        raise MemoryBudgetExceeded(
            f"searching below {limit} needs about {estimated} bytes of device memory "
            f"(budget {memory_budget_bytes}); use the chunked search"
        )
    if primes is not None and not primes.covers(math.isqrt(limit)):
        raise ValueError(f"prime list covers {primes.limit} but the search needs {math.isqrt(limit)}")
    return find_pairs(limit, primes=primes, device=device)
