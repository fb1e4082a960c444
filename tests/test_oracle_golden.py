"""Pins the CPU oracle (oracle/oracle.c) to the reference's own outputs.

The golden fixtures come from importing the unmodified reference
(tests/golden/make_golden.py); these tests run on CPU only.
"""
import hashlib
import math

import numpy as np
import pytest

from conftest import pair_keys


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def test_primes(orc, golden):
    for lim, rec in golden["primes"].items():
        if int(lim) > 2**21:
            continue
        p = orc.primes_up_to(int(lim))
        assert p.size == rec["count"] and digest(p) == rec["sha256"]


def test_sieve_small(orc, golden):
    p = orc.primes_up_to(2000)
    assert orc.sieve_segment(1, 10, p).tolist() == golden["sieve_small"]["1_10"]
    assert orc.sieve_segment(16, 1, p).tolist() == golden["sieve_small"]["16_1"]
    assert orc.sieve_segment(1213, 6, p).tolist() == golden["sieve_small"]["1213_6"]


def test_sieve_windows(orc, golden):
    for w in golden["sieve_windows"]:
        need = math.isqrt(w["start"] + w["length"] - 1)
        if need > 2**21:
            continue  # the 2^63 / 2^64 windows need multi-GB prime tables; GPU tests cover them
        vals = orc.sieve_segment(w["start"], w["length"], orc.primes_up_to(need), w["fast"])
        assert digest(vals) == w["sha256"], w["start"]


def test_trial_division(orc, golden):
    for rec in golden["trial_division"]:
        v = orc.radicals_trial_division(rec["start"], rec["length"])
        assert v[:8].tolist() == rec["head"] and digest(v) == rec["sha256"]


def test_strip_twos(orc, golden):
    v = np.arange(1, 1025, dtype=np.uint64)
    orc.strip_twos(v, 1)
    assert digest(v) == golden["strip_twos_1_1024_sha256"]
    assert v[39] == 10 and v[5] == 6 and v[1023] == 2


def test_hash(orc, golden):
    for lo, hi, size, slot in golden["commutative_hash"]:
        assert orc.slot_of(lo, hi, size - 1) == slot
    for c, size in golden["table_size_for"]:
        assert orc.table_size_for(c) == size
    for lim, s, n in golden["num_chunks"]:
        assert orc.num_chunks(lim, s) == n


def test_table_kernels(orc, golden):
    for t in golden["tables"]:
        rad_of = np.array(t["rad_of"], np.uint64)
        rad_next = np.array(t["rad_next"], np.uint64)
        built, inserted, slots = orc.build_table(t["start"], rad_of, rad_next, 2**64 - 1, t["table_size"])
        assert [list(r) for r in built] == t["built"]
        assert inserted == t["occupied"] and digest(slots) == t["slots_sha256"]
        probed = orc.probe_table(t["start"] - len(t["rad_of"]), rad_of, rad_next, t["start"], rad_of, rad_next, slots)
        assert [list(r) for r in probed] == t["probed"]


def test_brute_force(orc, golden):
    for lim, rows in golden["brute_force"].items():
        assert [list(r) for r in orc.brute_force(int(lim))] == rows


def test_find_pairs_sorted(orc, golden):
    for lim, rows in golden["find_pairs_sorted"].items():
        if int(lim) > 2**20:
            continue
        assert [list(r) for r in orc.find_pairs_sorted(int(lim))] == rows, lim


@pytest.mark.parametrize("case", ["1048576_4096", "20000_64", "5000_300"])
def test_run_full_chunked(orc, golden, case):
    limit, chunk = (int(x) for x in case.split("_"))
    assert [list(r) for r in orc.run_full_chunked(limit, chunk, threads=2)] == golden["run_full_chunked"][case]


def test_run_full_chunked_resume(orc, golden):
    got = [list(r) for r in orc.run_full_chunked(5000, 300, resume_from=8)]
    assert got == golden["run_full_chunked"]["5000_300_resume8"]


def test_known_solutions_small(orc, golden):
    exp = golden["expected_pairs_up_to"]["1048576"]
    got = orc.find_pairs_sorted(2**20)
    assert pair_keys(got) == pair_keys(exp["first"] + exp["second"])
