"""GPU parity: the sm_100a path against the reference's golden outputs and the C oracle.

Every test calls through the C ABI (libbenelux_b200.so via paper_2506_01099_b200._native).
Integer work, so the bar is bit-exact everywhere.
"""
import hashlib
import math

import numpy as np
import pytest

from conftest import pair_keys, rows_of

pytestmark = pytest.mark.gpu

bp = pytest.importorskip("paper_2506_01099_b200")


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


# ---------------------------------------------------------------- primes (a1) -------------
def test_primes_match_reference(golden):
    for lim, rec in golden["primes"].items():
        pl = bp.primes_up_to(int(lim))
        assert len(pl) == rec["count"], lim
        assert digest(pl.primes) == rec["sha256"], lim
        assert pl.limit == int(lim)


# ---------------------------------------------------------------- sieve (a2-a6) -----------
def test_sieve_small_vectors(golden):
    p2k = bp.primes_up_to(2000)
    assert bp.sieve_radicals(bp.Interval(1, 10), p2k).values.tolist() == golden["sieve_small"]["1_10"]
    assert bp.sieve_radicals(bp.Interval(16, 1), p2k).values.tolist() == golden["sieve_small"]["16_1"]
    seg = bp.sieve_radicals(bp.Interval.closed(1213, 1218), p2k)
    assert seg.values.tolist() == golden["sieve_small"]["1213_6"] == [1213, 1214, 15, 38, 1217, 1218]


@pytest.mark.parametrize("idx", range(12))
def test_sieve_windows(golden, idx):
    w = golden["sieve_windows"][idx]
    iv = bp.Interval(w["start"], w["length"])
    primes = bp.primes_up_to(bp.required_prime_bound(iv))
    vals = bp.sieve_radicals(iv, primes, ctz_fast_path=w["fast"]).values
    assert vals[:8].tolist() == w["head"]
    assert vals[-8:].tolist() == w["tail"]
    assert digest(vals) == w["sha256"]


def test_sieve_rejects_uncovered():
    with pytest.raises(ValueError):
        bp.sieve_radicals(bp.Interval(1, 1000), bp.primes_up_to(10))


def test_sieve_random_windows_vs_oracle(orc):
    rng = np.random.default_rng(20260811)
    for _ in range(40):
        start = int(rng.integers(1, 10**12))
        length = int(rng.integers(1, 300_000))
        fast = bool(rng.integers(0, 2))
        iv = bp.Interval(start, length)
        need = bp.required_prime_bound(iv)
        got = bp.sieve_radicals(iv, bp.primes_up_to(need), ctz_fast_path=fast).values
        want = orc.sieve_segment(start, length, orc.primes_up_to(need), fast)
        assert np.array_equal(got, want), (start, length, fast)


def test_sieve_large_window_vs_trial_division(orc):
    # a window spanning several segments and grid waves
    iv = bp.Interval(2**32 - 5_000_000, 12_000_000)
    got = bp.sieve_radicals(iv).values
    want = orc.sieve_segment(iv.start, iv.length, orc.primes_up_to(bp.required_prime_bound(iv)))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("variant", ["-1", "0", "1", "2"])
def test_sieve_narrow_slots_vs_oracle(orc, monkeypatch, variant):
    """Windows ending below 2^32 run the sieve with 32-bit shared-memory slots (BNX_SIEVE_NARROW
    picks the geometry, -1 the u64 kernel): windows at 1, ragged lengths, windows ending at
    2^32 - 1 and one crossing 2^32 (u64 slots), both ctz modes, against the oracle's sieve."""
    from paper_2506_01099_b200 import _native

    monkeypatch.setenv("BNX_SIEVE_NARROW", variant)
    ctx = _native.Context(0)
    try:
        rng = np.random.default_rng(int(variant) + 7)
        cases = [(1, 3 * 2**20 + 5), (2**32 - 2**21, 2**21), (2**32 - 1, 1), (2**32 - 2**20 + 3, 2**20 + 9)]
        cases += [(int(rng.integers(1, 2**32 - 2**20)), int(rng.integers(1, 2**20))) for _ in range(6)]
        for start, length in cases:
            for fast in (True, False):
                need = math.isqrt(start + length - 1)
                got = ctx.sieve_radicals(start, length, None, 0, fast)
                want = orc.sieve_segment(start, length, orc.primes_up_to(need + 1), fast)
                assert np.array_equal(got, want), (variant, start, length, fast)
    finally:
        ctx.close()


@pytest.mark.parametrize("gbuckets", ["0", "1"])
def test_sieve_global_buckets_vs_oracle(orc, monkeypatch, gbuckets):
    """Windows reaching 2^32 take the huge progressions' hits from one bucketing pass over the
    window (BNX_SIEVE_GBUCKETS=1, default) or scan them per segment (0): windows straddling
    2^32, at prime powers with large surpluses (3^22, 5^15, 2 * 7^13), random windows up to
    2^40, several segments and a ragged end, both ctz modes, against the oracle."""
    from paper_2506_01099_b200 import _native

    monkeypatch.setenv("BNX_SIEVE_GBUCKETS", gbuckets)
    ctx = _native.Context(0)
    try:
        rng = np.random.default_rng(int(gbuckets) + 11)
        cases = [(2**32 - 2**20 + 3, 2**21 + 9), (2**32, 5), (3**22 - 5000, 10001), (5**15 - 77, 300),
                 (2 * 7**13 - 3, 100), (2**36 - 2**19, 3 * 2**20 + 17)]
        cases += [(int(rng.integers(2**32, 2**40)), int(rng.integers(1, 2**21))) for _ in range(6)]
        for start, length in cases:
            for fast in (True, False):
                need = math.isqrt(start + length - 1)
                got = ctx.sieve_radicals(start, length, None, 0, fast)
                want = orc.sieve_segment(start, length, orc.primes_up_to(need + 1), fast)
                assert np.array_equal(got, want), (gbuckets, start, length, fast)
    finally:
        ctx.close()


def test_sieve_global_bucket_overflow_falls_back(orc, monkeypatch):
    """A global bucket that fills up (BNX_SIEVE_GCAP=1 forces it) makes the call re-run with
    the per-segment scan: same radicals as the oracle."""
    from paper_2506_01099_b200 import _native

    monkeypatch.setenv("BNX_SIEVE_GCAP", "1")
    ctx = _native.Context(0)
    try:
        for start, length in [(2**40 - 2**20, 2**21 + 3), (2**33 + 5, 3 * 2**19)]:
            got = ctx.sieve_radicals(start, length, None, 0, True)
            want = orc.sieve_segment(start, length, orc.primes_up_to(math.isqrt(start + length) + 1), True)
            assert np.array_equal(got, want), (start, length)
    finally:
        ctx.close()


# ---------------------------------------------------------------- trial division ---------
def test_trial_division_vectors(golden):
    for rec in golden["trial_division"]:
        v = bp.radicals_by_trial_division(bp.Interval(rec["start"], rec["length"]))
        assert v[:8].tolist() == rec["head"]
        assert digest(v) == rec["sha256"]


# ---------------------------------------------------------------- search (a7-a16) --------
@pytest.mark.parametrize("limit", ["3", "4", "10", "50", "517", "1300", "2000", "5000", "20000", "30000",
                                   "1000000", "1048576", "10000000", "16777216"])
def test_find_pairs_sorted_golden(golden, limit):
    got = rows_of(bp.find_pairs_sorted(int(limit)))
    assert got == golden["find_pairs_sorted"][limit]


def test_find_pairs_matches_brute_force_golden(golden):
    for lim, rows in golden["brute_force"].items():
        assert pair_keys(bp.find_pairs_sorted(int(lim))) == pair_keys(rows)


def test_all_limits_up_to_600_vs_oracle_brute_force(orc):
    for limit in range(3, 600):
        got = [tuple(r) for r in rows_of(bp.find_pairs_sorted(limit))]
        assert got == orc.brute_force(limit), limit


def test_random_limits_vs_oracle(orc):
    rng = np.random.default_rng(7)
    for limit in rng.integers(3, 3_000_000, 12).tolist():
        got = [tuple(r) for r in rows_of(bp.find_pairs_sorted(int(limit)))]
        assert got == orc.find_pairs_sorted(int(limit)), limit


@pytest.mark.parametrize("case", ["1048576_4096", "1048576_65536", "20000_64", "5000_300", "10000000_131072"])
def test_run_full_chunked_golden(golden, case):
    limit, chunk = (int(x) for x in case.split("_"))
    assert rows_of(bp.run_full_chunked(limit, chunk)) == golden["run_full_chunked"][case]


def test_run_full_chunked_resume_golden(golden):
    got = rows_of(bp.run_full_chunked(5000, 300, resume_from=8))
    assert got == golden["run_full_chunked"]["5000_300_resume8"]


def test_search_chunk_golden(golden):
    g = golden["search_chunk"]
    assert rows_of(bp.search_chunk(0, 1300, bp.primes_up_to(2000))) == g["0_1300_p2000"]
    assert rows_of(bp.search_chunk(0, 10001, bp.primes_up_to(101))) == g["0_10001_p101"]
    p = bp.primes_up_to(math.isqrt(bp.chunk_bounds(1, 1000).last))
    assert rows_of(bp.search_chunk(1, 1000, p)) == g["1_1000"]
    assert rows_of(bp.search_chunk(3, 100, bp.primes_up_to(2000))) == g["3_100_p2000"] == []
    assert rows_of(bp.search_chunk(1, 40000, bp.primes_up_to(300))) == g["1_40000_p300"]


def test_chunk_callback_order():
    events = []
    gen = bp.run_full_chunked(80_000, 1 << 12, on_chunk_done=lambda i: events.append(("done", i)))
    for pair in gen:
        events.append(("pair", pair.n))
    done = [e for e in events if e[0] == "done"]
    assert done == [("done", i) for i in range(bp.num_chunks(80_000, 1 << 12))]
    for pos, ev in enumerate(events):
        if ev[0] == "pair":
            boundary = next(i for kind, i in events[pos:] if kind == "done")
            assert ev[1] <= bp.chunk_bounds(boundary, 1 << 12).domain_last


@pytest.mark.parametrize("limit", ["1048576", "16777216", "10000000", "268435456", "4294967296"])
def test_known_solutions(golden, limit):
    exp = golden["expected_pairs_up_to"][limit]
    got = bp.find_pairs_sorted(int(limit), memory_budget_bytes=None)
    assert rows_of([p for p in got if p.kind == bp.Kind.FIRST]) == sorted(exp["first"], key=lambda r: (r[1], r[2]))
    assert rows_of([p for p in got if p.kind == bp.Kind.SECOND]) == sorted(exp["second"], key=lambda r: (r[1], r[2]))


def test_kind_filters_2p32(golden):
    exp = golden["expected_pairs_up_to"]["4294967296"]
    first = bp.find_pairs(2**32, kinds=bp.Kind.FIRST)
    second = bp.find_pairs(2**32, kinds=bp.Kind.SECOND)
    assert rows_of(first) == sorted(exp["first"], key=lambda r: (r[1], r[2]))
    assert rows_of(second) == sorted(exp["second"], key=lambda r: (r[1], r[2]))
    assert len(first) == 16 and len(second) == 17


def test_errors():
    with pytest.raises(ValueError):
        bp.find_pairs_sorted(2)
    with pytest.raises(bp.MemoryBudgetExceeded, match="chunked"):
        bp.find_pairs_sorted(10**6, memory_budget_bytes=10**6)
    # the reference's default budget (14 GiB at 48 B per record) refuses 2^32 as it does
    with pytest.raises(bp.MemoryBudgetExceeded):
        bp.find_pairs_sorted(2**32)
    assert len(bp.find_pairs_sorted(2**28)) == 29  # 48 * 2^28 = 12 GiB fits
    with pytest.raises(ValueError):
        list(bp.run_full_chunked(2, 300))
    with pytest.raises(ValueError):
        list(bp.run_full_chunked(5000, 2))


def test_reference_run_2p32_exact_rows():
    """The unmodified reference's own run_full_chunked(2^32, 2^28) (tests/golden/
    make_golden_2p32.py, 1430 s on 8 threads) against the device search: identical rows in
    identical (chunk, n, m) order."""
    import json
    import os

    from conftest import ROOT

    ref = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_pairs_2p32.json")))["rows"]
    assert rows_of(bp.run_full_chunked(2**32, 2**28)) == ref
    assert sorted(rows_of(bp.find_pairs_sorted(2**32, memory_budget_bytes=None)), key=lambda r: (r[1], r[2])) == \
        sorted(ref, key=lambda r: (r[1], r[2]))


class engine:
    """Switch the default context's candidate generator for a block (restores heavy)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        bp._native.context(None).set_engine(self.name)

    def __exit__(self, *exc):
        bp._native.context(None).set_engine("heavy")


def exact_candidates(orc, lo, hi):
    """#{lo <= n <= hi : rad(n) rad(n+1) <= 2n} from the oracle's sieve (numpy)."""
    vals = orc.sieve_segment(lo, hi - lo + 2, orc.primes_up_to(math.isqrt(hi + 1) + 1))
    n = np.arange(lo, hi + 1, dtype=np.uint64)
    r0, r1 = vals[:-1], vals[1:]
    return int(np.count_nonzero(r0 <= (2 * n) // r1))  # R <= 2n without overflow


@pytest.mark.parametrize("name", ["heavy", "screen"])
@pytest.mark.parametrize("e", [24, 28])
def test_generator_keeps_every_candidate(orc, e, name):
    """Both candidate generators may only over-approximate: the number of n < S with
    rad(n) rad(n+1) <= 2n that reach k_tail must equal the exact count from the oracle's
    sieve, i.e. no candidate is ever dropped (and, for the heavy generator, none is
    duplicated: it emits the candidates themselves)."""
    S = 1 << e
    exact = exact_candidates(orc, 1, S - 1)
    with engine(name):
        bp.find_pairs(S)
        st = bp.last_stats()
    assert st["candidates"] == exact
    assert st["survivors"] >= exact


def test_heavy_candidates_on_random_domains(orc):
    """Exact candidate count of the heavy generator on domains far from 1 (where most
    surplus classes have no heavy integer), against the oracle."""
    rng = np.random.default_rng(5)
    for _ in range(6):
        lo = int(rng.integers(1, 2**34))
        hi = lo + int(rng.integers(0, 1 << 22))
        bp.search_domain(lo, hi)
        assert bp.last_stats()["candidates"] == exact_candidates(orc, lo, hi), (lo, hi)


def test_heavy_candidates_beyond_the_paper(orc):
    """Windows between 2^42 and 2^48 (beyond the byte screen's range and the paper's 1.4e12):
    the heavy generator's exact candidate count equals the oracle's sieve count."""
    rng = np.random.default_rng(9)
    for top in (44, 46, 48):
        lo = int(rng.integers(2**(top - 2), 2**top - 2**22))
        hi = lo + (1 << 21)
        bp.search_domain(lo, hi)
        assert bp.last_stats()["candidates"] == exact_candidates(orc, lo, hi), (lo, hi)


def test_heavy_boundaries(orc):
    """Domains where the heavy generator switches arithmetic (neighbours below / above 2^32:
    32-bit tests vs residues), single-integer domains and the very start: exact candidate
    counts against the oracle and identical rows to the byte screen."""
    cases = [(2**32 - 2**20, 2**32 + 2**20), (2**32 - 3, 2**32 + 3), (1, 1), (1, 2), (2, 2), (3, 8),
             (1214, 1216), (2**33 + 7, 2**33 + 7)]
    for lo, hi in cases:
        rows = {}
        for name in ("heavy", "screen"):
            with engine(name):
                rows[name] = np.ascontiguousarray(bp.search.search_rows(lo, hi)).tobytes()
                cand = bp.last_stats()["candidates"]
                if hi - lo < 2**22:
                    assert cand == exact_candidates(orc, lo, hi), (name, lo, hi)
        assert rows["heavy"] == rows["screen"], (lo, hi)


@pytest.mark.parametrize("lo,hi", [(1, 2**32 - 1), (2**32, 2**33 - 1), (2**40 - 2**30, 2**40 - 1),
                                   (1_400_000_000_000 - 2**28, 1_400_000_000_000), (2**42 - 2**26, 2**42 - 2)])
def test_engines_agree(lo, hi):
    """The heavy generator and the byte screen return identical rows and candidate counts."""
    out = {}
    for name in ("heavy", "screen"):
        with engine(name):
            rows = bp.search.search_rows(lo, hi)
            out[name] = (np.ascontiguousarray(rows).tobytes(), bp.last_stats()["candidates"])
    assert out["heavy"] == out["screen"]


def test_whole_range_to_2p40_is_theorem_1():
    """One device search over [1, 2^40) (both kinds): exactly the 41 pairs of Theorem 1."""
    S = 1 << 40
    from oracle import theorem1

    got = sorted((p.m, p.n) for p in bp.find_pairs(S))
    assert got == theorem1.known_pairs(S)
    assert len(got) == 41


def test_random_domains_vs_oracle(orc):
    rng = np.random.default_rng(11)
    for _ in range(10):
        lo = int(rng.integers(1, 2_000_000))
        hi = lo + int(rng.integers(0, 1_000_000))
        got = [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in bp.search_domain(lo, hi)]
        want = sorted((r for r in orc.find_pairs_sorted(hi + 1) if r[2] >= lo), key=lambda r: (r[2], r[1]))
        assert got == want, (lo, hi)


def test_near_the_top_of_the_range():
    """Largest supported bounds: the first-kind family member (2^k - 2, 2^(2k) - 2^(k+1)) just
    below the top must be found with its radicals -- k = 24 below 2^48 with the heavy
    generator, k = 21 below 2^42 with the byte screen -- and larger bounds are refused."""
    for name, k, top in (("heavy", 24, 2**48), ("screen", 21, 2**42)):
        with engine(name):
            m, n = 2**k - 2, 2**(2 * k) - 2**(k + 1)
            got = bp.search_domain(n - 5000, n + 5000)
            assert [(int(p.kind), p.m, p.n) for p in got] == [(1, m, n)], name
            p = got[0]
            assert (p.rad_m, p.rad_m_plus_1) == (bp.radical_oracle(m), bp.radical_oracle(m + 1))
            with pytest.raises(ValueError):
                bp.search_domain(top - 10, top + 1)


@pytest.mark.parametrize("name", ["heavy", "screen"])
def test_shards_partition_the_search(name):
    """bnx_ctx_set_shard: the shards of one search return disjoint row sets whose union is
    the full search (heavy: item shards; screen: n-slabs), for several shard counts."""
    ctx = bp._native.context(None)
    lo, hi = 1, 2**32 - 1
    with engine(name):
        full = sorted(map(tuple, bp.search.search_rows(lo, hi).tolist()))
        try:
            for nsh in (2, 3, 7):
                parts = []
                for sh in range(nsh):
                    ctx.set_shard(sh, nsh)
                    parts += list(map(tuple, bp.search.search_rows(lo, hi).tolist()))
                assert sorted(parts) == full, nsh
        finally:
            ctx.set_shard(0, 1)
    with pytest.raises(ValueError):
        ctx.set_shard(3, 3)


def test_repeated_searches_are_identical():
    """Back-to-back device searches (the bench's pattern) give identical rows and counters:
    guards the CTA-level work queue of k_heavy_screen against barrier/race bugs."""
    ctx = bp._native.context(None)
    ctx.prepare(2**32)
    ctx.enqueue(1, 2**32 - 1, 3)
    ref = np.ascontiguousarray(ctx.collect()).tobytes()
    ref_st = ctx.stats()
    for _ in range(300):
        ctx.enqueue(1, 2**32 - 1, 3)
        assert np.ascontiguousarray(ctx.collect()).tobytes() == ref
        st = ctx.stats()
        assert (st["survivors"], st["candidates"], st["matches"]) == \
            (ref_st["survivors"], ref_st["candidates"], ref_st["matches"])


# ------------------------------------------- BASELINE configs[3] / configs[4] at full size ----
def _rows(pairs):
    return [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs]


def test_paper_range_both_kinds_is_theorem_1():
    """configs[4]: every pair of both kinds below 1.4e12 in one device search -- exactly the
    42 rows of Theorem 1, radicals included."""
    from oracle import theorem1

    S = theorem1.COMPLETENESS_BOUND
    want = theorem1.known_rows(S)
    assert len(want) == 42
    assert _rows(bp.find_pairs_sorted(S, memory_budget_bytes=None)) == want
    for kind in (1, 2):
        got = _rows(bp.search.find_pairs(S, kinds=kind))
        assert got == [r for r in want if r[0] == kind], kind


@pytest.mark.parametrize("nshards", [2, 4, 8])
def test_multi_gpu_shards_paper_range(nshards):
    """configs[3]/[4] through the multi-device entry point (bnx_search_multi): `nshards`
    item shards (here all on cuda:0) below 2^40 (first kind) and below 1.4e12 (both kinds)
    merge to exactly Theorem 1."""
    from oracle import theorem1

    S40 = 1 << 40
    got = _rows(bp.find_pairs_multi_gpu(S40, [0] * nshards, kinds=1))
    assert got == [r for r in theorem1.known_rows(S40) if r[0] == 1]
    assert len(got) == 20
    S = theorem1.COMPLETENESS_BOUND
    assert _rows(bp.find_pairs_multi_gpu(S, [0] * nshards)) == theorem1.known_rows(S)


def test_item_shards_strong_config_partition():
    """configs[3]'s per-rank work (bench.py --gpus N): the 8 item shards of the first-kind
    search below 2^40 are disjoint and their union is the unsharded search."""
    ctx = bp._native.context(None)
    full = sorted(map(tuple, bp.search.search_rows(1, 2**40 - 1, kinds=1).tolist()))
    parts = []
    try:
        for sh in range(8):
            ctx.set_shard(sh, 8)
            parts += list(map(tuple, bp.search.search_rows(1, 2**40 - 1, kinds=1).tolist()))
    finally:
        ctx.set_shard(0, 1)
    assert sorted(parts) == full and len(full) == 20


@pytest.mark.parametrize("kmin", [1, 64, 256])
def test_sieve_mask_mode_at_small_bounds(orc, monkeypatch, kmin):
    """k_heavy_sieve's mask mode (at most 64 primes below P2: bounds up to ~2^33) forced onto
    every class with >= kmin k (BNX_HEAVY_KMIN, read when a context is created): exact
    candidate counts against the oracle's sieve, the same rows as the default split, on
    domains with 32-bit and wider y, and the 2^32 search's survivor list is unchanged."""
    from paper_2506_01099_b200 import _native

    base = _native.context(0)
    monkeypatch.setenv("BNX_HEAVY_KMIN", str(kmin))
    ctx = _native.Context(0)
    try:
        for lo, hi in [(1, 2**22), (2**32 - 2**21, 2**32 + 2**21), (2**33 - 2**20, 2**33), (5, 5)]:
            got = ctx.search_domain(lo, hi, 3, None, 0)
            assert ctx.stats()["candidates"] == exact_candidates(orc, lo, hi), (kmin, lo, hi)
            want = base.search_domain(lo, hi, 3, None, 0)
            assert got.tobytes() == want.tobytes(), (kmin, lo, hi)
        got = ctx.search(2**32, 3, None, 0)
        st = ctx.stats()
        want = base.search(2**32, 3, None, 0)
        assert got.tobytes() == want.tobytes()
        assert st["survivors"] == base.stats()["survivors"] and st["candidates"] == 2253
    finally:
        ctx.close()


@pytest.mark.parametrize("mode", ["0", "1"])
def test_exact_stage_modes(orc, monkeypatch, mode):
    """k_heavy_exact one thread per survivor (0: every prime from P2 to cbrt y) or one warp per
    survivor (1: only the primes that can complete a p^2 q factor large enough), each forced
    on both sides of the default switch: exact candidate counts against the oracle's sieve
    and the same rows as the default context, near 2^32, 2^40, 1.4e12 and 2^46, and the
    whole 2^32 search."""
    from paper_2506_01099_b200 import _native

    base = _native.context(0)
    monkeypatch.setenv("BNX_EXACT_WARP", mode)
    ctx = _native.Context(0)
    try:
        for lo, hi in [(1, 2**22), (2**32 - 2**21, 2**32 + 2**21), (2**40 - 2**21, 2**40 - 1),
                       (1_400_000_000_000 - 2**21, 1_400_000_000_000), (2**46 - 2**20, 2**46 - 2)]:
            got = ctx.search_domain(lo, hi, 3, None, 0)
            assert ctx.stats()["candidates"] == exact_candidates(orc, lo, hi), (mode, lo, hi)
            assert got.tobytes() == base.search_domain(lo, hi, 3, None, 0).tobytes(), (mode, lo, hi)
        got = ctx.search(2**32, 3, None, 0)
        assert got.tobytes() == base.search(2**32, 3, None, 0).tobytes()
        assert ctx.stats()["candidates"] == 2253
    finally:
        ctx.close()


@pytest.mark.gpu
def test_local_tile_scan_matches_cub_scan(monkeypatch):
    """Below ~2^33 (no sieve classes) the class counts are scanned per tile of 256 and the
    screen adds the tile offsets itself; BNX_LOCAL_SCAN=0 keeps the cub scan.  Same rows and
    counters either way, from bounds with an odd number of stage-1 primes up to 2^32."""
    from paper_2506_01099_b200 import _native

    base = _native.context(0)
    monkeypatch.setenv("BNX_LOCAL_SCAN", "0")
    ctx = _native.Context(0)
    try:
        keys = ("survivors", "candidates", "residue_checks", "matches", "pairs")
        for lo, hi in [(1, 1000), (1, 2**20), (3, 2**26 + 12345), (2**31 - 2**22, 2**31 + 2**22),
                       (2**32 - 2**21, 2**32 - 1), (1, 2**32 - 1), (5, 2**33)]:
            for kinds in (1, 3):
                a = base.search_domain(lo, hi, kinds, None, 0)
                sa = base.stats()
                b = ctx.search_domain(lo, hi, kinds, None, 0)
                sb = ctx.stats()
                assert a.tobytes() == b.tobytes(), (lo, hi, kinds)
                assert {k: sa[k] for k in keys} == {k: sb[k] for k in keys}, (lo, hi, kinds)
    finally:
        ctx.close()
