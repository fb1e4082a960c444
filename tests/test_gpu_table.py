"""The paper's Algorithm 3 on the GPU (paper_2506_01099_b200.table) against the reference's
SignatureTable / build_table / probe_table / search_chunk outputs."""
import numpy as np
import pytest

from conftest import pair_keys, rows_of

pytestmark = pytest.mark.gpu
bp = pytest.importorskip("paper_2506_01099_b200")


def test_table_kernels_golden(golden):
    for t in golden["tables"]:
        rad_of = np.array(t["rad_of"], np.uint64)
        rad_next = np.array(t["rad_next"], np.uint64)
        tab = bp.SignatureTable(t["start"], rad_of, rad_next)
        assert tab.table_size == t["table_size"]
        built = tab.insert_all()
        assert tab.occupied == t["occupied"]
        # the reference's serial discovery order: a build meets the stored entries of one
        # signature in insertion order along the probe chain, i.e. (n, m); a probe (m, n)
        assert rows_of(built) == t["built"]
        probed = tab.probe_all(t["start"] - len(t["rad_of"]), rad_of, rad_next)
        assert rows_of(probed) == t["probed"]
        # probe paths have no holes and every entry stays in the domain (test_chunked.py:203-218)
        slots = tab.slots
        size = tab.table_size
        for idx in np.flatnonzero(slots):
            packed = int(slots[idx])
            home, off = packed & 0xFFFFFFFF, (packed >> 32) - 1
            assert 0 <= off < len(t["rad_of"])
            walk = home
            while walk != idx:
                assert slots[walk] != 0
                walk = (walk + 1) % size


def test_table_full_raises():
    vals = bp.sieve_radicals(bp.Interval(1, 1300)).values
    tab = bp.SignatureTable(1, vals[:11], vals[1:12], table_size=8)
    with pytest.raises(bp.TableFullError):
        tab.insert_all()


def test_insert_respects_n_limit():
    vals = bp.sieve_radicals(bp.Interval(1, 1300)).values
    tab = bp.SignatureTable(1, vals[:-1], vals[1:])
    tab.insert_all(n_limit=100)
    assert tab.occupied == 99


def test_search_chunk_table_golden(golden):
    g = golden["search_chunk"]
    assert rows_of(bp.search_chunk_table(0, 1300)) == g["0_1300_p2000"]
    assert rows_of(bp.search_chunk_table(0, 10001)) == g["0_10001_p101"]
    assert rows_of(bp.search_chunk_table(1, 1000)) == g["1_1000"]
    assert rows_of(bp.search_chunk_table(3, 100)) == []
    assert rows_of(bp.search_chunk_table(1, 40000)) == g["1_40000_p300"]


@pytest.mark.parametrize("case", ["1048576_4096", "1048576_65536", "20000_64", "5000_300"])
def test_run_full_chunked_table_golden(golden, case):
    limit, chunk = (int(x) for x in case.split("_"))
    assert rows_of(bp.run_full_chunked_table(limit, chunk)) == golden["run_full_chunked"][case]


def test_algorithm3_equals_residue_search_2p26():
    a = pair_keys(bp.run_full_chunked_table(1 << 26, 1 << 22))
    b = pair_keys(bp.find_pairs_sorted(1 << 26))
    assert a == b and len(a) == 27
