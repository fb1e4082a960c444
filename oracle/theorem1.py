"""Theorem 1 of the paper as a checker: every Benelux pair below 1.4e12.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py): used by tests/, __graft_entry__.smoke()
and bench.py to check the device search at bounds no CPU search reaches.  Never imported by
the product package.

PAPER.md:257-273 (Theorem 1) states that below 1.4e12 the pairs are exactly
  * first kind:  (2^k - 2, 2^k (2^k - 2)) for k >= 2, and (75, 1215);
  * second kind: (2^k + 1, 2^k (2^k + 2)) for k >= 0, and (35, 4374).
The reference ships the same list as pkg/src/benelux_pairs/families.py:17-107
(family_first_kind / family_second_kind / exceptional_pairs / expected_pairs_up_to); this
module derives it from the closed forms and re-verifies every row with an exact radical
(Miller-Rabin + Pollard-Brent factorisation), so each row carries rad(m) and rad(m+1) and a
wrong closed form would fail loudly.  The identity behind the families:
  first:  m = 2(2^(k-1) - 1), n = 2^(k+1)(2^(k-1) - 1):   rad m = rad n,
          m + 1 = 2^k - 1, n + 1 = (2^k - 1)^2:            rad(m+1) = rad(n+1);
  second: m = 2^k + 1, n + 1 = (2^k + 1)^2:                rad m = rad(n+1),
          m + 1 = 2(2^(k-1) + 1), n = 2^(k+1)(2^(k-1) + 1): rad(m+1) = rad n  (k >= 1; k = 0 gives (2, 3)).
"""
from __future__ import annotations

import math
import random

COMPLETENESS_BOUND = 1_400_000_000_000
EXCEPTIONAL = ((1, 75, 1215), (2, 35, 4374))  # PAPER.md:265-268 (kind, m, n)


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:  # deterministic for n < 3.3e24
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _factor(n: int, out: set) -> None:
    if n == 1:
        return
    if _is_prime(n):
        out.add(n)
        return
    for p in (2, 3, 5, 7, 11, 13):
        if n % p == 0:
            out.add(p)
            while n % p == 0:
                n //= p
            _factor(n, out)
            return
    rng = random.Random(n)
    while True:  # Pollard-Brent
        y, c, m = rng.randrange(1, n), rng.randrange(1, n), 64
        g, r, q = 1, 1, 1
        while g == 1:
            x = y
            for _ in range(r):
                y = (y * y + c) % n
            k = 0
            while k < r and g == 1:
                ys = y
                for _ in range(min(m, r - k)):
                    y = (y * y + c) % n
                    q = q * abs(x - y) % n
                g = math.gcd(q, n)
                k += m
            r *= 2
        if g == n:
            g = 1
            while g == 1:
                ys = (ys * ys + c) % n
                g = math.gcd(abs(x - ys), n)
        if g != n:
            _factor(g, out)
            _factor(n // g, out)
            return


def radical(n: int) -> int:
    """rad(n): the product of the distinct primes dividing n (rad(1) = 1)."""
    if n < 1:
        raise ValueError("radical of a non-positive integer")
    primes: set = set()
    _factor(n, primes)
    return math.prod(primes)


def _row(kind: int, m: int, n: int) -> tuple[int, int, int, int, int]:
    rm, rm1, rn, rn1 = radical(m), radical(m + 1), radical(n), radical(n + 1)
    ok = (rm, rm1) == (rn, rn1) if kind == 1 else (rm, rm1) == (rn1, rn)
    if not ok or not 0 < m < n:
        raise AssertionError(f"({m}, {n}) is not a pair of kind {kind}")
    return kind, m, n, rm, rm1


def first_kind_member(k: int) -> tuple[int, int]:
    """(2^k - 2, 2^k (2^k - 2)), k >= 2."""
    if k < 2:
        raise ValueError("the first-kind family starts at k = 2")
    return (1 << k) - 2, (1 << k) * ((1 << k) - 2)


def second_kind_member(k: int) -> tuple[int, int]:
    """(2^k + 1, 2^k (2^k + 2)), k >= 0."""
    if k < 0:
        raise ValueError("the second-kind family starts at k = 0")
    return (1 << k) + 1, (1 << k) * ((1 << k) + 2)


def known_rows(limit: int, *, beyond_bound: bool = False) -> list[tuple[int, int, int, int, int]]:
    """Rows (kind, m, n, rad m, rad m+1) of every pair with n < limit, sorted by (m, n).
    Complete (Theorem 1) for limit <= 1.4e12; `beyond_bound` lists the families and the two
    exceptional pairs past it (then a search may legitimately find more)."""
    if limit > COMPLETENESS_BOUND and not beyond_bound:
        raise ValueError(f"Theorem 1 covers n < {COMPLETENESS_BOUND}; got limit {limit}")
    rows = []
    for kind, member, k0 in ((1, first_kind_member, 2), (2, second_kind_member, 0)):
        k = k0
        while True:
            m, n = member(k)
            if n >= limit:
                break
            rows.append(_row(kind, m, n))
            k += 1
    rows += [_row(kind, m, n) for kind, m, n in EXCEPTIONAL if n < limit]
    return sorted(rows, key=lambda r: (r[1], r[2]))


def known_pairs(limit: int, kind: int | None = None, **kw) -> list[tuple[int, int]]:
    """(m, n) of the rows of `kind` (1, 2, or None for both), sorted by (m, n)."""
    return [(r[1], r[2]) for r in known_rows(limit, **kw) if kind is None or r[0] == kind]
