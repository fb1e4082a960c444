"""How much of k_heavy_exact's trial division a survivor really needs (CPU analysis).

For the stage-1 survivors of a window [lo, hi] searched with the bound S (numpy + the oracle
sieve, restating y_tests: odd primes <= P2 divided out, U(c) as surplus_bound), the exact
stage only has to find a p^2 q factor with p >= t, t = c / (2n / (rad x rad_small(y))): the
primes in [max(t, p1), cbrt c) or [p1, c / max(t, p1)^2].  Prints the class shares and the
mean primes to try per survivor (and per warp of 32, the max) against the full np3.

    python scripts/exact_ranges.py 40 30     # window of 2^30 below 2^40
"""
import bisect
import math
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), ".."))
from oracle import oracle  # noqa: E402


def icbrt(v):
    r = round(v ** (1 / 3))
    while r ** 3 > v:
        r -= 1
    while (r + 1) ** 3 <= v:
        r += 1
    return r


def main():
    e, w = int(sys.argv[1]), int(sys.argv[2])
    S = 1 << e
    hi, lo = S - 1, S - (1 << w)
    y_max = hi + 2
    p2 = math.isqrt(math.isqrt(y_max))
    primes = [int(p) for p in oracle.primes_up_to(1 << 22)]
    odd = primes[1:]
    np2 = (sum(1 for p in odd if p <= p2) + 31) // 32 * 32
    small = odd[:np2]
    p1 = odd[np2]
    cb = icbrt(y_max)
    np3 = sum(1 for p in odd if p <= cb)
    sp = oracle.primes_up_to(math.isqrt(hi + 2) + 1)
    stats = {"reject_B": 0, "full": 0, "sqcube": 0, "cut": 0}
    blocks = []  # (t, blocks needed) of the cut survivors
    work, surv = [], 0
    step = 1 << 24
    for base in range(lo, hi + 1, step):
        ln = min(step, hi + 1 - base)
        rad = oracle.sieve_segment(base, ln, sp).astype(np.uint64)
        x = np.arange(base, base + ln, dtype=np.uint64)
        sig = x // rad
        heavy = np.nonzero(2 * sig.astype(np.float64) ** 2 >= x.astype(np.float64))[0]
        for i in heavy:
            xv, sv = int(x[i]), int(sig[i])
            if 2 * sv * sv < xv:
                continue
            for side in (0, 1):
                y = xv - 1 if side else xv + 1
                if side and (xv < 2 or y < 1):
                    continue
                tz = (y & -y).bit_length() - 1
                c, sy, rs = y >> tz, (1 << (tz - 1)) if tz else 1, 2 if tz else 1
                for p in small:
                    if c % p == 0:
                        rs *= p
                        c //= p
                        while c % p == 0:
                            c //= p
                            sy *= p
                u = 1
                if c >= p1 * p1:
                    q = math.isqrt(c)
                    if q * q == c:
                        u = q
                    if c >= p1 ** 3:
                        u = max(u, math.isqrt(c // p1) + 1)
                        r = icbrt(c)
                        if r ** 3 == c:
                            u = max(u, r * r)
                if 2 * sv * sy * u < (xv if side else xv + 1):
                    continue
                surv += 1
                n = y if side else xv
                B = (2 * n) // (xv // sv) // rs
                if B == 0:
                    stats["reject_B"] += 1
                    work.append(0)
                    continue
                t = -(-c // B)
                if t <= 1:
                    stats["full"] += 1
                    work.append(np3)
                    continue
                q = math.isqrt(c)
                r = icbrt(c)
                if q * q == c or r ** 3 == c:
                    stats["sqcube"] += 1
                    work.append(0)
                    continue
                stats["cut"] += 1
                tp = max(t, p1)
                top = icbrt(c)
                if tp > top:
                    stats["tau_above_cbrt"] = stats.get("tau_above_cbrt", 0) + 1
                    hb = min(top, c // (tp * tp))
                    stats["sum_ratio_hiB_top"] = stats.get("sum_ratio_hiB_top", 0.0) + hb / top
                lo_b, hi_b = p1, min(top, c // (tp * tp))
                lo_a, hi_a = tp, top - 1
                # 32-prime blocks (from index np2) a lane needs
                ib = bisect.bisect_right(odd, hi_b)
                ia0, ia1 = bisect.bisect_left(odd, lo_a), bisect.bisect_right(odd, top)
                need = set(range(np2 // 32, (ib + 31) // 32)) | set(range(ia0 // 32, (ia1 + 31) // 32))
                blocks.append((tau_of := t, need))
                segs = sorted(s for s in ((lo_a, hi_a), (lo_b, hi_b)) if s[0] <= s[1])
                cnt, cur = 0, 0
                for a, b in segs:
                    a = max(a, cur + 1)
                    if a <= b:
                        cnt += bisect.bisect_right(odd, b) - bisect.bisect_left(odd, a)
                        cur = b
                work.append(cnt)
    wk = np.array(work, dtype=np.float64)
    rng = np.random.default_rng(0)
    perm = rng.permutation(len(wk))
    warps = wk[perm][: len(wk) // 32 * 32].reshape(-1, 32).max(axis=1) if len(wk) >= 32 else wk
    # the same warps after sorting each group of 256 survivors (one CTA) by its range
    g = wk[perm][: len(wk) // 256 * 256].reshape(-1, 256) if len(wk) >= 256 else wk[perm].reshape(1, -1)
    gs = np.sort(g, axis=1)
    sorted_max = gs[:, : gs.shape[1] // 32 * 32].reshape(-1, 32).max(axis=1) if gs.shape[1] >= 32 else gs.max(axis=1)
    # warps iterating the global blocks, skipping a block no lane needs: after sorting each
    # group of 256 by t, the blocks a warp runs (union of its lanes) against all of np2..np3
    nb_all = (np3 + 31) // 32 - np2 // 32
    order = rng.permutation(len(blocks))
    bl = [blocks[i] for i in order]
    unions = []
    for g0 in range(0, len(bl) - 255, 256):
        grp = sorted(bl[g0:g0 + 256], key=lambda r: r[0])
        for w0 in range(0, 256, 32):
            u = set()
            for _, nd in grp[w0:w0 + 32]:
                u |= nd
            unions.append(len(u))
    print({"blocks_all": nb_all, "warp_union_sorted": round(float(np.mean(unions)), 2) if unions else None})
    print({"S": f"2^{e}", "window": f"2^{w}", "survivors": surv, **stats, "np2": np2, "np3": np3,
           "mean_primes": round(float(wk.mean()), 1) if len(wk) else 0,
           "mean_warp_max": round(float(warps.mean()), 1) if len(wk) else 0,
           "mean_warp_max_sorted256": round(float(sorted_max.mean()), 1) if len(wk) else 0})


if __name__ == "__main__":
    main()
