"""Generate the golden fixtures in tests/golden/golden.json from the UNMODIFIED reference.

Imports the reference package in place (/root/reference/pkg/src) and
records its outputs on the inputs the parity tests use.  Run from the repo root:
    python tests/golden/make_golden.py
The JSON is committed; the tests never read /root/reference.
Large windows are stored as a sha256 of the little-endian uint64 array plus head/tail values.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import benelux_pairs as bp  # noqa: E402
from benelux_pairs import _kernels  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def rows(pairs):
    return [[int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1] for p in pairs]


def window(start: int, length: int, fast: bool = True) -> dict:
    iv = bp.Interval(start, length)
    primes = bp.primes_up_to(bp.required_prime_bound(iv))
    vals = bp.sieve_radicals(iv, primes, ctz_fast_path=fast).values
    return {
        "start": start, "length": length, "fast": fast, "sha256": digest(vals),
        "head": [int(v) for v in vals[:8]], "tail": [int(v) for v in vals[-8:]],
    }


def main() -> None:
    g: dict = {}
    # --- primes (primes.py:24-35) ------------------------------------------------------
    g["primes"] = {
        str(lim): {"count": len(bp.primes_up_to(lim)), "sha256": digest(bp.primes_up_to(lim).primes)}
        for lim in (0, 1, 2, 10, 2000, 65536, math.isqrt(2**40), math.isqrt(1_400_000_000_000))
    }
    # --- sieve windows (radical.py:109-124, _kernels.py:48-84) -------------------------
    small = {
        "1_10": bp.sieve_radicals(bp.Interval(1, 10), bp.primes_up_to(2000)).values.tolist(),
        "16_1": bp.sieve_radicals(bp.Interval(16, 1), bp.primes_up_to(2000)).values.tolist(),
        "1213_6": bp.sieve_radicals(bp.Interval.closed(1213, 1218), bp.primes_up_to(2000)).values.tolist(),
    }
    g["sieve_small"] = small
    wins = [
        (1, 1_000_000, True), (1, 1_000_000, False), (10**9, 100_001, True), (10**9, 100_001, False),
        (2**32 - 2**16, 2**17, True), (2**40 - 2**14, 2**15, True),
        (1_400_000_000_000 - 2**14, 2**15, True), (2**63, 4097, True), (2**64 - 4097, 4096, True),
        (123_456_789, 777, True), (1, 1, True), (2, 3, False),
    ]
    g["sieve_windows"] = [window(s, n, f) for s, n, f in wins]
    # --- trial division oracle (_kernels.py:87-112) ------------------------------------
    td = []
    for s, n in ((1, 100_000), (10**9, 4000), (2**40 - 500, 1000), (1_400_000_000_000 - 64, 128)):
        v = bp.radicals_by_trial_division(bp.Interval(s, n))
        td.append({"start": s, "length": n, "sha256": digest(v), "head": v[:8].tolist()})
    g["trial_division"] = td
    # --- strip twos (_kernels.py:33-45) ------------------------------------------------
    seg = bp.strip_twos_fast(bp.fresh_segment(bp.Interval(1, 1024)))
    g["strip_twos_1_1024_sha256"] = digest(seg.values)
    # --- hash (chunked.py:93-109) ------------------------------------------------------
    rng = np.random.default_rng(20260811)
    hv = []
    for _ in range(64):
        a, b = (int(x) for x in rng.integers(1, 2**62, 2))
        lo, hi = min(a, b), max(a, b) + 1
        for size in (64, 4096, 1 << 29):
            hv.append([lo, hi, size, bp.commutative_hash(bp.PairSignature(lo, hi), size)])
    g["commutative_hash"] = hv
    g["table_size_for"] = [[c, bp.table_size_for(c)] for c in (1, 2, 3, 7, 100, 2**24 - 1, 2**27 - 1)]
    g["num_chunks"] = [[l, s, bp.num_chunks(l, s)] for l, s in ((3, 3), (5000, 300), (2**20, 2**12), (2**32, 2**27), (2**40, 2**27), (1_400_000_000_000, 2**27))]
    # --- table kernels on small-pool signatures (test_chunked.py:169-199) ---------------
    tables = []
    for seed in (1, 7, 20260811):
        r = np.random.default_rng(seed)
        count = int(r.integers(2, 400))
        rad_of = r.integers(1, 40, count).astype(np.uint64)
        rad_next = rad_of + r.integers(1, 40, count).astype(np.uint64)
        start = int(r.integers(count + 1, 2**40))
        t = bp.SignatureTable(start, rad_of, rad_next)
        built = t.insert_all()
        probed = t.probe_all(start - count, rad_of, rad_next)
        tables.append({
            "seed": seed, "start": start, "rad_of": rad_of.tolist(), "rad_next": rad_next.tolist(),
            "table_size": t.table_size, "occupied": t.occupied, "slots_sha256": digest(t.slots),
            "built": rows(built), "probed": rows(probed),
        })
    g["tables"] = tables
    # --- pair lists ---------------------------------------------------------------------
    g["brute_force"] = {str(l): rows(bp.brute_force_pairs(l)) for l in (3, 10, 1300, 5000, 20000)}
    g["find_pairs_sorted"] = {
        str(l): rows(bp.find_pairs_sorted(l))
        for l in (3, 4, 10, 50, 517, 1300, 2000, 5000, 20000, 30000, 10**6, 2**20, 10**7, 2**24)
    }
    g["run_full_chunked"] = {
        "1048576_4096": rows(bp.run_full_chunked(2**20, 2**12)),
        "1048576_65536": rows(bp.run_full_chunked(2**20, 2**16)),
        "20000_64": rows(bp.run_full_chunked(20000, 64)),
        "5000_300": rows(bp.run_full_chunked(5000, 300)),
        "5000_300_resume8": rows(bp.run_full_chunked(5000, 300, resume_from=8)),
        "10000000_131072": rows(bp.run_full_chunked(10**7, 2**17, threads=os.cpu_count() or 1)),
    }
    g["search_chunk"] = {
        "0_1300_p2000": rows(bp.search_chunk(0, 1300, bp.primes_up_to(2000))),
        "0_10001_p101": rows(bp.search_chunk(0, 10001, bp.primes_up_to(101))),
        "1_1000": rows(bp.search_chunk(1, 1000, bp.primes_up_to(math.isqrt(bp.chunk_bounds(1, 1000).last)))),
        "3_100_p2000": rows(bp.search_chunk(3, 100, bp.primes_up_to(2000))),
        "1_40000_p300": rows(bp.search_chunk(1, 40000, bp.primes_up_to(300))),
    }
    exp = {}
    for lim in (2**20, 2**24, 10**7, 2**28, 2**32, 2**40, 1_400_000_000_000):
        ks = bp.expected_pairs_up_to(lim)
        exp[str(lim)] = {"first": rows(ks.first_kind), "second": rows(ks.second_kind)}
    g["expected_pairs_up_to"] = exp
    g["brute_force_scan_small"] = list(_kernels.brute_force_scan(
        bp.radicals_by_trial_division(bp.Interval(1, 10)), np.zeros(8, np.int8),
        np.zeros(8, np.uint64), np.zeros(8, np.uint64))[:1])
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote golden.json")


if __name__ == "__main__":
    main()
