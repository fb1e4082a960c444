"""Property tests of the host-side formats and types (CPU): CLI row formats and checkpoint
text round-trip, the fast row conversion equals the dataclass constructor, the reference-type
conversion, the Theorem 1 checker's closed forms."""
import numpy as np
from hypothesis import given, strategies as st

from paper_2506_01099_b200 import cli, signatures as sg
from paper_2506_01099_b200._native import PAIR_DTYPE

u63 = st.integers(min_value=1, max_value=(1 << 63) - 1)
rows = st.lists(st.tuples(st.sampled_from([1, 2]), u63, u63, u63, u63), max_size=20)


@given(rows, st.sampled_from(["csv", "jsonl"]))
def test_row_format_round_trip(tmp_path_factory, rs, fmt):
    f = cli.RowFormat(fmt)
    path = tmp_path_factory.mktemp("rows") / f"r.{fmt}"
    path.write_text(f.header + "".join(f.encode(r) for r in rs))
    assert f.read(str(path)) == [tuple(r) for r in rs]


@given(st.integers(0, 2**64), st.integers(3, 2**40), st.integers(0, 2**40))
def test_checkpoint_round_trip(limit, chunk, nxt):
    p = cli.Progress(limit, chunk, nxt)
    assert cli.Progress.from_text(p.text()) == p


@given(st.lists(st.tuples(u63, u63, u63, u63, st.sampled_from([1, 2])), max_size=30))
def test_fast_rows_equal_the_constructor(rs):
    arr = np.zeros(len(rs), dtype=PAIR_DTYPE)
    good = []
    for i, (m, n, rm, rm1, k) in enumerate(rs):
        m, n = min(m, n), max(m, n)
        if m == n:
            n += 1
        arr[i] = (m, n, rm, rm1, k, 0)
        good.append(sg.BeneluxPair(m, n, sg.Kind(k), rm, rm1))
    got = sg.pairs_from_rows(arr)
    assert got == good and all(type(p) is sg.BeneluxPair for p in got)


def test_fast_rows_keep_the_invariant():
    arr = np.zeros(1, dtype=PAIR_DTYPE)
    arr[0] = (5, 5, 1, 1, 1, 0)
    try:
        sg.pairs_from_rows(arr)
    except ValueError:
        return
    raise AssertionError("m == n must be refused")


def test_to_reference_types():
    class RefKind(int):
        pass

    class RefPair:
        def __init__(self, m, n, kind, rm, rm1):
            self.t = (m, n, kind, rm, rm1)

    p = sg.BeneluxPair(75, 1215, sg.Kind.FIRST, 15, 38)
    (r,) = sg.to_reference([p], RefPair, RefKind)
    assert r.t == (75, 1215, 1, 15, 38) and type(r.t[2]) is RefKind


@given(st.integers(2, 24), st.integers(0, 24))
def test_theorem1_members_are_pairs(k1, k2):
    from oracle import theorem1

    m, n = theorem1.first_kind_member(k1)
    assert theorem1._row(1, m, n)[0] == 1
    m, n = theorem1.second_kind_member(k2)
    assert theorem1._row(2, m, n)[0] == 2
