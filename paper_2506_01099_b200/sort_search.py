"""Full search below a bound -- drop-in for the reference's ``sort_search.py``.

``find_pairs_sorted`` keeps the reference's signature, result (every pair m < n < limit, both
kinds, sorted by (m, n); sort_search.py:37-91) and failure modes, including the memory-budget
refusal (sort_search.py:53-58: 48 bytes per record, 14 GiB default, MemoryBudgetExceeded
pointing to the chunked search), so code written against the reference behaves the same.  The
B200 engine itself keeps nothing per integer: ``memory_budget_bytes=None`` lifts the refusal
(every bound up to 2^48), and ``find_pairs`` is the same search without the reference's
budget rule.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from .primes import PrimeList
from .radical import RadicalSegment
from .search import find_pairs
from .signatures import BeneluxPair, PairSignature, signature_of

# values + lo + hi + sort order + two sorted key copies, all uint64 (sort_search.py:17-19)
BYTES_PER_RECORD = 48
DEFAULT_MEMORY_BUDGET = 14 * 2**30


class MemoryBudgetExceeded(ValueError):
    """The search would not fit the memory budget; use the chunked search."""


@dataclass(frozen=True)
class SignatureRecord:
    n: int
    sig: PairSignature


def signature_record(n: int, segment: RadicalSegment) -> SignatureRecord:
    """Record (n, signature of n) read off a radical segment."""
    return SignatureRecord(n, signature_of(n, segment.rad(n), segment.rad(n + 1)))


def find_pairs_sorted(limit: int, primes: PrimeList | None = None, *,
                      memory_budget_bytes: int | None = DEFAULT_MEMORY_BUDGET, device: int | None = None
                      ) -> list[BeneluxPair]:
    """Every Benelux pair of either kind with m < n < limit, sorted by (m, n)."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    estimated = BYTES_PER_RECORD * limit
    if memory_budget_bytes is not None and estimated > memory_budget_bytes:
        raise MemoryBudgetExceeded(
            f"sorting {limit} records needs about {estimated} bytes "
            f"(budget {memory_budget_bytes}); use the chunked search"
        )
    if primes is not None and not primes.covers(math.isqrt(limit)):
        raise ValueError(f"prime list covers {primes.limit} but the search needs {math.isqrt(limit)}")
    return find_pairs(limit, primes=primes, device=device)
