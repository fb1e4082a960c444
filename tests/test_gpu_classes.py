"""The heavy generator's surplus-class table, built on the device (csrc/bnx_classes.cu), must
equal the host depth-first search it replaces -- the same classes (b, m, r) in the same order
(k_heavy_screen's speed depends on the order)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

bp = pytest.importorskip("paper_2506_01099_b200")


def dfs_classes(X: int):
    """The DFS of the round-1 host builder (bnx_capi.cu build_heavy_host), in Python:
    every powerful b <= X with m = sigma / r, r = rad(b), in DFS order."""
    root = math.isqrt(X)
    sieve = bytearray([1]) * (root + 1)
    sieve[:2] = b"\x00\x00"[: min(2, root + 1)]
    for i in range(2, math.isqrt(root) + 1):
        if sieve[i]:
            sieve[i * i::i] = bytearray(len(sieve[i * i::i]))
    P = [i for i in range(root + 1) if sieve[i]]
    out = []
    stack = [(1, 1, 1, 0)]  # (b, sigma, r, next prime index)
    while stack:
        b, sigma, r, nxt = stack.pop()
        out.append((b, sigma // r, r))
        for i in range(nxt, len(P)):
            p = P[i]
            if b > X // (p * p):
                break
            cb, cs = b * p * p, sigma * p
            while True:
                stack.append((cb, cs, r * p, i + 1))
                if cb > X // p:
                    break
                cb *= p
                cs *= p
    return out


@pytest.mark.parametrize("X", [3, 4, 100, 65_536, 10**6 + 7, 2**32, 2**34 + 12345])
def test_device_class_table_is_the_host_dfs(X):
    ctx = bp._native.Context(0)
    try:
        b, mr = ctx.class_table(X)
    finally:
        ctx.close()
    want = dfs_classes(X)
    assert len(b) == len(want)
    assert np.array_equal(b, np.array([w[0] for w in want], np.uint64))
    assert np.array_equal(mr & np.uint64((1 << 40) - 1), np.array([w[1] for w in want], np.uint64))
    assert np.array_equal(mr >> np.uint64(40), np.array([w[2] for w in want], np.uint64))


def test_class_count_at_the_paper_bound():
    """Count at 1.4e12 against the powerful-number count (every b <= X is u^2 v^3 exactly once)."""
    X = 1_400_000_000_000
    ctx = bp._native.Context(0)
    try:
        b, _ = ctx.class_table(X)
    finally:
        ctx.close()
    V = round(X ** (1 / 3)) + 2
    mu2 = np.ones(V + 1, bool)
    for p in range(2, math.isqrt(V) + 1):
        mu2[p * p::p * p] = False
    want = sum(math.isqrt(X // (v ** 3)) for v in range(1, V + 1) if mu2[v] and v ** 3 <= X)
    assert len(b) == want
    assert len(np.unique(b)) == len(b) and int(b.max()) <= X
