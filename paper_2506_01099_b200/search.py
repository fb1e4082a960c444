"""The B200 search engine: every Benelux pair with n in a domain, on one GPU.

The whole path runs on the device (csrc/bnx_heavy.cu, csrc/bnx_kernels.cu):
  k_heavy_count -> scan -> k_heavy_screen -> k_heavy_exact -> k_tail -> k_tail_heavy
and the host only receives the (tiny) verified pair list.  See DESIGN.md for the lemma
(rad(n) rad(n+1) <= 2n for every pair) that lets the collision pass work per n without
materialising any per-integer record.
"""
from __future__ import annotations

from . import _native
from .primes import PrimeList
from .signatures import BeneluxPair, Kind, pairs_from_rows


def kinds_mask(kinds) -> int:
    """None / "both" -> both kinds; Kind.FIRST / 1 / "first"; Kind.SECOND / 2 / "second"."""
    if kinds is None or kinds == "both" or kinds == 3:
        return _native.KIND_BOTH
    if kinds in (Kind.FIRST, 1, "first"):
        return _native.KIND_FIRST
    if kinds in (Kind.SECOND, 2, "second"):
        return _native.KIND_SECOND
    raise ValueError(f"unknown kind selector {kinds!r}")


def _prime_args(primes: PrimeList | None):
    if primes is None:
        return None, 0
    return primes.primes, primes.limit


def search_rows(n_first: int, n_last: int, *, kinds=None, primes: PrimeList | None = None,
                device: int | None = None):
    """Raw bnx_pair_t rows for every pair with n_first <= n <= n_last, sorted by (n, m)."""
    if n_first < 1 or n_last < n_first:
        raise ValueError("empty search domain")
    p, lim = _prime_args(primes)
    return _native.context(device).search_domain(n_first, n_last, kinds_mask(kinds), p, lim)


def search_domain(n_first: int, n_last: int, *, kinds=None, primes: PrimeList | None = None,
                  device: int | None = None) -> list[BeneluxPair]:
    """BeneluxPair list for n_first <= n <= n_last (any m < n), sorted by (n, m)."""
    return pairs_from_rows(search_rows(n_first, n_last, kinds=kinds, primes=primes, device=device))


def find_pairs(limit: int, *, kinds=None, primes: PrimeList | None = None,
               device: int | None = None) -> list[BeneluxPair]:
    """Every pair m < n < limit of the selected kinds, sorted by (m, n)."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    p, lim = _prime_args(primes)
    rows = _native.context(device).search(limit, kinds_mask(kinds), p, lim)
    return pairs_from_rows(rows)


def last_stats(device: int | None = None) -> dict:
    """Counters of the last search on `device` (survivors, candidates, matches, ...)."""
    return _native.context(device).stats()


def find_pairs_multi_gpu(limit: int, devices, *, kinds=None, primes: PrimeList | None = None) -> list[BeneluxPair]:
    """Every pair m < n < limit on several GPUs driven from this thread (bnx_search_multi):
    device i computes shard i of len(devices); the merged list equals find_pairs(limit)."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    p, lim = _prime_args(primes)
    return pairs_from_rows(_native.search_multi(list(devices), limit, kinds_mask(kinds), p, lim))
