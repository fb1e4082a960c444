"""Quadratic reference search on the GPU (mirror of the reference's bruteforce.py:16-42).

Trial-division radicals plus the all-pairs scan (k_trial_division + k_brute_force); shares
nothing with the screen / residue-class search, so the self-test can pit the two against
each other.  Practical up to ~10^6 (limited to 2^22)."""
from __future__ import annotations

from . import _native
from .signatures import BeneluxPair, pairs_from_rows


def brute_force_pairs(limit: int, *, device: int | None = None) -> list[BeneluxPair]:
    """All pairs of either kind with m < n < limit, sorted by (m, n)."""
    if limit < 3:
        raise ValueError("limit must be >= 3")
    return pairs_from_rows(_native.context(device).brute_force(limit))
