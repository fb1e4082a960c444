"""Host-side logic (no GPU): reference-mirroring types and geometry, the sharding maths, the
chunk streaming of run_full_chunked, and the number theory the device search relies on,
checked against the reference's golden outputs and the C oracle."""
import math

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_2506_01099_b200 as bp
from paper_2506_01099_b200 import _native, chunked, dist
from conftest import pair_keys, rows_of


# ---------------------------------------------------------------- types & geometry -------
def test_interval_validation():
    assert bp.Interval(5, 3).last == 7
    assert bp.Interval.closed(1213, 1218) == bp.Interval(1213, 6)
    for start, length in [(0, 5), (1, 0), (2**64 - 1, 2)]:
        with pytest.raises(ValueError):
            bp.Interval(start, length)
    assert bp.required_prime_bound(bp.Interval(1, 1000)) == 31


def test_signatures_and_classify():
    assert bp.signature_of(75, 15, 38) == bp.PairSignature(15, 38) == bp.signature_of(1215, 38, 15)
    assert bp.compare(bp.PairSignature(2, 3), bp.PairSignature(2, 5)) == -1
    assert bp.compare(bp.PairSignature(15, 38), bp.PairSignature(15, 38)) == 0
    assert bp.classify(75, 1215, 15, 38, 15, 38) == bp.BeneluxPair(75, 1215, bp.Kind.FIRST, 15, 38)
    assert bp.classify(35, 4374, 35, 6, 6, 35) == bp.BeneluxPair(35, 4374, bp.Kind.SECOND, 35, 6)
    assert bp.classify(3, 5, 3, 2, 5, 6) is None
    with pytest.raises(ValueError):
        bp.classify(5, 3, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        bp.BeneluxPair(3, 3, bp.Kind.FIRST, 1, 1)


def test_chunk_geometry_matches_reference(golden):
    c = bp.chunk_bounds(1, 5)
    assert (c.first, c.last, c.domain_first, c.domain_last) == (5, 9, 5, 8)
    for count, size in golden["table_size_for"]:
        assert bp.table_size_for(count) == size
    for limit, s, n in golden["num_chunks"]:
        assert bp.num_chunks(limit, s) == n
    for lo, hi, size, slot in golden["commutative_hash"]:
        assert bp.commutative_hash(bp.PairSignature(lo, hi), size) == slot
    with pytest.raises(ValueError):
        bp.commutative_hash(bp.PairSignature(1, 2), 1000)


def test_host_helpers_match_reference(golden):
    import hashlib

    seg = bp.strip_twos_fast(bp.fresh_segment(bp.Interval(1, 1024)))
    digest = hashlib.sha256(np.ascontiguousarray(seg.values, dtype="<u8").tobytes()).hexdigest()
    assert digest == golden["strip_twos_1_1024_sha256"]
    assert seg.rad(40) == 10 and seg.rad(6) == 6 and seg.rad(1024) == 2
    assert [bp.radical_oracle(n) for n in (1, 75, 1216, 1218)] == [1, 15, 38, 1218]


@pytest.mark.parametrize("limit", ["1048576", "16777216", "10000000", "268435456", "4294967296", "1099511627776",
                                   "1400000000000"])
def test_theorem1_oracle_matches_reference(golden, limit):
    """oracle/theorem1.py (the checker used beyond CPU-search range) against the reference's
    own expected_pairs_up_to rows (families.py:77-107), radicals included."""
    from oracle import theorem1

    exp = golden["expected_pairs_up_to"][limit]
    got = theorem1.known_rows(int(limit))
    assert [list(r) for r in got if r[0] == 1] == sorted(exp["first"], key=lambda r: (r[1], r[2]))
    assert [list(r) for r in got if r[0] == 2] == sorted(exp["second"], key=lambda r: (r[1], r[2]))


# ---------------------------------------------------------------- the lemma -----------------
def _rows(golden_rows):
    return [tuple(r) for r in golden_rows]


def test_every_reference_pair_satisfies_the_key_bound(golden):
    """rad(n) rad(n+1) <= 2n for every pair (Lemma 1), on all reference outputs,
    and R | n - m (first kind) or R | n + m + 1 (second kind)."""
    rows = set()
    for lim, rs in golden["find_pairs_sorted"].items():
        rows |= set(_rows(rs))
    for k in golden["expected_pairs_up_to"].values():
        rows |= set(_rows(k["first"] + k["second"]))
    assert len(rows) > 40
    for kind, m, n, rm, rm1 in rows:
        rn, rn1 = (rm, rm1) if kind == 1 else (rm1, rm)
        R = rn * rn1
        assert R <= 2 * n
        assert (n - m) % R == 0 if kind == 1 else (n + m + 1) % R == 0


def _rad(x):
    return bp.radical_oracle(x)


def residue_search(limit):
    """Pure-Python model of the device algorithm (k_screen's exact condition, k_tail's
    residue classes and radical checks) for small limits."""
    out = []
    rads = [0] + [_rad(x) for x in range(1, limit + 1)]
    for n in range(1, limit):
        r0, r1 = rads[n], rads[n + 1]
        R = r0 * r1
        if R > 2 * n:
            continue
        t = 1
        while n - t * R >= 1:
            m = n - t * R
            if rads[m] == r0 and rads[m + 1] == r1:
                out.append((1, m, n, r0, r1))
            t += 1
        t = (n + 1) // R + 1
        while t * R <= 2 * n:
            m = t * R - n - 1
            if rads[m] == r1 and rads[m + 1] == r0:
                out.append((2, m, n, r1, r0))
            t += 1
    return sorted(out, key=lambda r: (r[1], r[2]))


@pytest.mark.parametrize("limit", [3, 4, 10, 517, 1300, 5000, 20000])
def test_residue_model_equals_reference(golden, limit):
    key = str(limit)
    want = golden["find_pairs_sorted"].get(key) or golden["brute_force"][key]
    assert [list(r) for r in residue_search(limit)] == want


def test_residue_model_equals_oracle_brute_force(orc):
    for limit in range(3, 400):
        assert residue_search(limit) == orc.brute_force(limit)


def test_log_screen_threshold_is_conservative():
    """The screen keeps n iff sum of half-bit weights >= floor(2 log2(n+1)) - 2; check that
    every n with rad(n) rad(n+1) <= 2n passes with the exact device weights (CPU model)."""
    limit = 200_000
    wt = {}

    def weight(p):
        if p not in wt:
            wt[p] = 2 if p == 2 else math.ceil(2 * math.log2(p) + 1e-7)
        return wt[p]

    def A(x):
        a, y, p = 0, x, 2
        while p * p <= y:
            e = 0
            while y % p == 0:
                y //= p
                e += 1
            if e >= 2:
                a += (e - 1) * weight(p)
            p += 1
        return a

    def floor2log2(v):
        e = v.bit_length() - 1
        return 2 * e + (v * v >= 2 ** (2 * e + 1))

    for n in range(1, limit):
        if _rad(n) * _rad(n + 1) <= 2 * n:
            assert A(n) + A(n + 1) >= max(0, floor2log2(n + 1) - 2), n


# ---------------------------------------------------------------- sharding / streaming ---
@given(st.integers(1, 10**12), st.integers(0, 10**6), st.integers(1, 9))
@settings(max_examples=60)
def test_shards_tile_the_domain(first, span, world):
    last = first + span
    pieces = [dist.shard_domain(first, last, r, world) for r in range(world)]
    covered = [p for p in pieces if p]
    assert covered[0][0] == first and covered[-1][1] == last
    for a, b in zip(covered, covered[1:]):
        assert b[0] == a[1] + 1
    sizes = [p[1] - p[0] + 1 for p in covered]
    assert max(sizes) - min(sizes) <= 1


def test_weak_shards():
    assert dist.weak_shard(2**32, 0, 1) == (1, 2**32 - 1)
    assert dist.weak_shard(100, 0, 3) == (1, 100)
    assert dist.weak_shard(100, 1, 3) == (101, 200)
    assert dist.weak_shard(100, 2, 3) == (201, 299)


def _oracle_rows(orc, lo, hi):
    rows = [r for r in orc.find_pairs_sorted(hi + 1) if lo <= r[2] <= hi]
    rows.sort(key=lambda r: (r[2], r[1]))
    arr = np.zeros(len(rows), dtype=_native.PAIR_DTYPE)
    for i, (k, m, n, rm, rm1) in enumerate(rows):
        arr[i] = (m, n, rm, rm1, k, 0)
    return arr


def test_run_full_chunked_streaming_logic(orc, monkeypatch, golden):
    """run_full_chunked's batching/splitting/callbacks with the device search replaced by
    the oracle (the GPU tests cover the real path)."""
    calls = []

    def fake(lo, hi, **kw):
        calls.append((lo, hi))
        return _oracle_rows(orc, lo, hi)

    monkeypatch.setattr(chunked, "search_rows", fake)
    monkeypatch.setattr(chunked, "_prepare_run", lambda *a: None)
    monkeypatch.setattr(chunked, "BATCH_INTEGERS", 50_000)
    for case in ("1048576_4096", "20000_64", "5000_300"):
        limit, s = (int(x) for x in case.split("_"))
        events = []
        got = []
        for p in bp.run_full_chunked(limit, s, on_chunk_done=lambda i: events.append(i)):
            got.append(p)
        assert rows_of(got) == golden["run_full_chunked"][case]
        assert events == list(range(bp.num_chunks(limit, s)))
    assert len(calls) > 3  # batched into several device searches
    assert rows_of(bp.run_full_chunked(5000, 300, resume_from=8)) == golden["run_full_chunked"]["5000_300_resume8"]
    assert list(bp.run_full_chunked(5000, 300, resume_from=bp.num_chunks(5000, 300))) == []


def test_search_chunk_domain_logic(orc, monkeypatch, golden):
    monkeypatch.setattr(chunked, "search_rows", lambda lo, hi, **kw: _oracle_rows(orc, lo, hi))
    g = golden["search_chunk"]
    assert rows_of(bp.search_chunk(0, 1300, bp.PrimeList(np.array([2, 3], np.uint64), 2000))) == g["0_1300_p2000"]
    assert rows_of(bp.search_chunk(3, 100, None)) == []
    with pytest.raises(ValueError):
        bp.search_chunk(5, 1000, bp.PrimeList(np.array([2], np.uint64), 10))
    assert bp.search_chunk(0, 100, None, n_limit=1) == []


def test_reference_2p32_fixture_is_theorem_1(golden):
    import json
    import os

    from conftest import ROOT

    ref = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_pairs_2p32.json")))["rows"]
    exp = golden["expected_pairs_up_to"]["4294967296"]
    assert sorted(map(tuple, ref)) == sorted(map(tuple, exp["first"] + exp["second"]))
