"""Raw C ABI on the GPU: the status-code protocol (_kernels.py:17-19 semantics), the
split-phase API, stream attachment and the device-memory sieve."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
_native = pytest.importorskip("paper_2506_01099_b200._native")


@pytest.fixture(scope="module")
def L():
    return _native.load()


@pytest.fixture(scope="module")
def ctx(L):
    h = ctypes.c_void_p()
    assert L.bnx_ctx_create(0, ctypes.byref(h)) == _native.BNX_OK
    yield h
    L.bnx_ctx_destroy(h)


def test_buffer_full_protocol(L, ctx, golden):
    found = ctypes.c_size_t(0)
    small = (_native.PairRow * 4)()
    st = L.bnx_search(ctx, 2**32, 3, None, 0, 0, small, 4, ctypes.byref(found))
    assert st == _native.BNX_BUFFER_FULL and found.value == 33
    big = (_native.PairRow * found.value)()
    assert L.bnx_search(ctx, 2**32, 3, None, 0, 0, big, found.value, ctypes.byref(found)) == _native.BNX_OK
    rows = [[r.kind, r.m, r.n, r.rad_m, r.rad_m1] for r in big]
    exp = golden["expected_pairs_up_to"]["4294967296"]
    assert rows == sorted(exp["first"] + exp["second"], key=lambda r: (r[1], r[2]))


def test_error_codes(L, ctx):
    found = ctypes.c_size_t(0)
    buf = (_native.PairRow * 4)()
    assert L.bnx_search(ctx, 2, 3, None, 0, 0, buf, 4, ctypes.byref(found)) == _native.BNX_ERR_INVALID
    assert L.bnx_search(ctx, 100, 0, None, 0, 0, buf, 4, ctypes.byref(found)) == _native.BNX_ERR_INVALID
    assert L.bnx_search(ctx, (1 << 48) + 1, 3, None, 0, 0, buf, 4, ctypes.byref(found)) == _native.BNX_ERR_RANGE
    assert L.bnx_ctx_set_shard(ctx, 2, 2) == _native.BNX_ERR_INVALID
    assert L.bnx_ctx_set_shard(ctx, 0, 0) == _native.BNX_ERR_INVALID
    primes = np.array([2, 3, 5, 7], np.uint64)
    p = primes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    assert L.bnx_search(ctx, 10**6, 3, p, 4, 10, buf, 4, ctypes.byref(found)) == _native.BNX_ERR_PRIMES_UNCOVERED
    assert b"covers" in L.bnx_last_error()
    out = np.empty(10, np.uint64)
    assert L.bnx_sieve_radicals(ctx, 0, 10, None, 0, 0, 1, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))) \
        == _native.BNX_ERR_INVALID


def test_split_phase_and_stats():
    ctx = _native.Context(0)
    try:
        ctx.set_timing(True)
        ctx.prepare(2**32)
        ctx.enqueue(1, 2**32 - 1, 1)
        rows = ctx.collect()
        assert len(rows) == 16 and all(int(k) == 1 for k in rows["kind"])
        st = ctx.stats()
        assert st["integers"] == 2**32 - 1 and st["pairs"] == 16 and st["candidates"] >= 16
        screen_ms, pipe_ms = ctx.timing()
        assert 0 < screen_ms <= pipe_ms
        with pytest.raises(ValueError):
            ctx.enqueue(1, 2**33, 1)  # not prepared that far
    finally:
        ctx.close()


def test_torch_stream_and_device_sieve():
    torch = pytest.importorskip("torch")
    ctx = _native.Context(0)
    try:
        s = torch.cuda.Stream()
        ctx.set_stream(s.cuda_stream)
        out = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
        with torch.cuda.stream(s):
            ctx.sieve_radicals_dev(1, out.numel(), out.data_ptr())
        s.synchronize()
        from oracle import oracle as orc

        want = orc.sieve_segment(1, 1 << 20, orc.primes_up_to(1024))
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want)
    finally:
        ctx.close()


@pytest.mark.parametrize("ctz", [True, False])
@pytest.mark.parametrize("start,length", [(987654321, (1 << 20) + 12345), (3, 777), (2**40 - 5, 70_001)])
def test_device_sieve_unaligned_output(start, length, ctz):
    """bnx_sieve_radicals_dev into a pointer that is 8- but not 16-byte aligned (a tensor
    view at an odd element offset): every tile of every segment must still be initialised
    (the 16-byte store path is skipped), ragged lengths included."""
    torch = pytest.importorskip("torch")
    from oracle import oracle as orc
    import paper_2506_01099_b200 as pkg

    ctx = _native.Context(0)
    try:
        buf = torch.full((length + 2,), -1, dtype=torch.int64, device="cuda")
        ctx.sieve_radicals_dev(start, length, buf.data_ptr() + 8, ctz_fast_path=ctz)
        torch.cuda.synchronize()
        got = buf.cpu().numpy().view(np.uint64)
        iv = pkg.Interval(start, length)
        want = orc.sieve_segment(start, length, orc.primes_up_to(pkg.required_prime_bound(iv)))
        assert np.array_equal(got[1 : length + 1], want)
        assert got[0] == np.uint64(2**64 - 1) and got[length + 1] == np.uint64(2**64 - 1)  # no stray writes
        with pytest.raises(ValueError, match="aligned"):
            ctx.sieve_radicals_dev(start, 16, buf.data_ptr() + 4)
    finally:
        ctx.close()


def test_domain_search_equals_filtered_full(L, ctx):
    found = ctypes.c_size_t(0)
    buf = (_native.PairRow * 64)()
    assert L.bnx_search_domain(ctx, 1000, 5_000_000, 3, None, 0, 0, buf, 64, ctypes.byref(found)) == 0
    dom = [(r.m, r.n) for r in buf[: found.value]]
    assert L.bnx_search(ctx, 5_000_001, 3, None, 0, 0, buf, 64, ctypes.byref(found)) == 0
    full = sorted(((r.m, r.n) for r in buf[: found.value] if r.n >= 1000), key=lambda x: (x[1], x[0]))
    assert dom == full


def test_engine_selection(L, ctx):
    """bnx_ctx_set_engine / bnx_ctx_engine: both generators through the C ABI, same rows;
    unknown engines are rejected with BNX_ERR_INVALID and leave the engine unchanged."""
    assert L.bnx_ctx_engine(ctx) == 0  # heavy by default
    found = ctypes.c_size_t(0)
    rows = {}
    for eng in (1, 0):
        assert L.bnx_ctx_set_engine(ctx, eng) == 0
        assert L.bnx_ctx_engine(ctx) == eng
        buf = (_native.PairRow * 64)()
        assert L.bnx_search(ctx, 1 << 24, 3, None, 0, 0, buf, 64, ctypes.byref(found)) == 0
        rows[eng] = [(r.m, r.n, r.rad_m, r.rad_m1, r.kind) for r in buf[: found.value]]
    assert rows[0] == rows[1] and len(rows[0]) == 25
    assert L.bnx_ctx_set_engine(ctx, 7) == 4
    assert L.bnx_ctx_engine(ctx) == 0


def test_graph_replay_follows_parameter_changes():
    """The heavy engine replays its search as CUDA graphs: changing the domain, the kinds,
    the stream or the timing switch must re-capture (same rows as a fresh context), and a
    repeat must replay with identical rows and counters."""
    import torch

    c = _native.Context(0)
    try:
        want = {}
        fresh = _native.Context(0)
        try:
            for lo, hi, kinds in ((1, 2**24, 3), (5_000_000, 2**24, 1), (1, 2**24, 2)):
                want[(lo, hi, kinds)] = fresh.search_domain(lo, hi, kinds, None, 0).tobytes()
        finally:
            fresh.close()
        s = torch.cuda.Stream()
        for timing in (False, True):
            c.set_timing(timing)
            for stream in (0, s.cuda_stream):
                c.set_stream(stream)
                for key, rows in want.items():
                    for _ in range(2):
                        assert c.search_domain(key[0], key[1], key[2], None, 0).tobytes() == rows
        c.set_stream(0)
    finally:
        c.close()


@pytest.mark.parametrize("prefix", ["0", "5"])
def test_rows_beyond_the_read_back_prefix(prefix, golden):
    """collect() returns the rows from the read-back copy when a search has at most
    PAIR_PREFIX pairs, else with a second copy; a context started with a smaller prefix
    (BNX_PAIR_PREFIX) takes the second path for the 33 pairs below 2^32."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = ("import json; from paper_2506_01099_b200 import _native; c = _native.Context(0); "
            "r = c.search(2**32, 3, None, 0); print(json.dumps([[int(x['kind']), int(x['m']), int(x['n']), "
            "int(x['rad_m']), int(x['rad_m1'])] for x in r]))")
    env = dict(os.environ, BNX_PAIR_PREFIX=prefix)
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    exp = golden["expected_pairs_up_to"]["4294967296"]
    assert json.loads(out.stdout.strip().splitlines()[-1]) == sorted(exp["first"] + exp["second"],
                                                                      key=lambda r: (r[1], r[2]))


def test_smallest_limits_with_a_caller_prime_list(golden):
    """limit 3 (isqrt = 1: the supplied list covers it with no primes at all) returns the
    reference's empty result instead of failing in the table build; 4 and 10 stay golden."""
    import paper_2506_01099_b200 as bp

    rows = lambda ps: [[int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1] for p in ps]  # noqa: E731
    assert bp.find_pairs_sorted(3, bp.primes_up_to(1)) == [] == golden["find_pairs_sorted"]["3"]
    assert rows(bp.find_pairs_sorted(4, bp.primes_up_to(2))) == golden["find_pairs_sorted"]["4"]
    with pytest.raises(ValueError):  # isqrt(4) = 2 is not covered by the primes up to 1
        bp.find_pairs_sorted(4, bp.primes_up_to(1))
    assert [(int(p.kind), p.m, p.n) for p in bp.find_pairs_sorted(10, bp.primes_up_to(3))] == \
        [(2, 2, 3), (1, 2, 8), (2, 3, 8)]
    assert bp.search_chunk(0, 3, bp.primes_up_to(1), n_limit=3) == []
    assert list(bp.run_full_chunked(3, 3, bp.primes_up_to(1))) == []


def test_collect_keeps_rows_after_buffer_full():
    """bnx_search_collect answering BNX_BUFFER_FULL keeps the rows: the retry with a large
    enough buffer returns them (no 'no search enqueued')."""
    L = _native.load()
    ctx = _native.Context(0)
    try:
        ctx.prepare(2**32)
        ctx.enqueue(1, 2**32 - 1, 3)
        found = ctypes.c_size_t(0)
        small = (_native.PairRow * 2)()
        assert L.bnx_search_collect(ctx.handle, small, 2, ctypes.byref(found)) == _native.BNX_BUFFER_FULL
        assert found.value == 33
        big = (_native.PairRow * 33)()
        assert L.bnx_search_collect(ctx.handle, big, 33, ctypes.byref(found)) == _native.BNX_OK
        assert found.value == 33 and sorted((r.m, r.n) for r in big)[0] == (2, 3)
    finally:
        ctx.close()


def test_table_search_chunk_refuses_oversized_tables():
    """chunk_size - 1 > 2^30 would need more than 2^32 slots (32-bit home slots); refused
    like the reference's SignatureTable (chunked.py:157-158) instead of dropping pairs."""
    import paper_2506_01099_b200 as bp

    with pytest.raises(ValueError):
        bp.search_chunk_table(0, (1 << 30) + 2)
    L = _native.load()
    ctx = _native.context(0)
    found = ctypes.c_size_t(0)
    buf = (_native.PairRow * 4)()
    assert L.bnx_table_search_chunk(ctx.handle, 0, (1 << 30) + 2, 2**40, 0, 0, buf, 4,
                                    ctypes.byref(found)) == _native.BNX_ERR_INVALID


def test_c_program_through_the_abi(tmp_path, golden):
    """examples/search_c.c, compiled with gcc against include/benelux_b200.h and linked to the
    library, prints the reference CLI's rows for every pair below 2^32."""
    import os
    import subprocess

    from conftest import ROOT

    exe = str(tmp_path / "search_c")
    lib = os.path.join(ROOT, "paper_2506_01099_b200")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "search_c.c"),
                    "-L", lib, "-lbenelux_b200", f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    out = subprocess.run([exe, str(2**32)], capture_output=True, text=True, check=True).stdout
    exp = golden["expected_pairs_up_to"]["4294967296"]
    want = sorted(exp["first"] + exp["second"], key=lambda r: (r[1], r[2]))
    assert out == "kind,m,n,rad_m,rad_m1\n" + "".join(",".join(map(str, r)) + "\n" for r in want)


def test_graph_cache_eviction_keeps_results():
    """More distinct searches than the context's graph cache holds (8), twice over: every
    replayed or re-captured graph returns the same rows as the first time."""
    import paper_2506_01099_b200 as bp

    domains = [(1 + 7 * i, 2**24 + 99991 * i) for i in range(11)]
    first = [np.ascontiguousarray(bp.search.search_rows(lo, hi)).tobytes() for lo, hi in domains]
    again = [np.ascontiguousarray(bp.search.search_rows(lo, hi)).tobytes() for lo, hi in reversed(domains)]
    assert first == list(reversed(again))
