"""Small workloads over every device engine, for compute-sanitizer runs.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python scripts/sanitize.py

(compute-sanitizer is closed on this round's GPU pool; the script runs plain there, and
the oracle comparisons below are the check.)

The workloads the oracle (oracle/, the CPU restatement) finishes fast are checked against
it, so a run also fails loudly on a wrong answer; the window near 2^40 is only exercised.  Sizes are small: the sanitizer serialises and
instruments every access.  Covered: the heavy generator (k_heavy_count, cub scan,
k_heavy_screen, k_heavy_exact, k_tail, k_tail_heavy), the heavy sieve (a window near
2^40), the byte-screen engine, the exact sieve into host and device buffers, and the
signature table build/probe."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_01099_b200 as pkg  # noqa: E402
from paper_2506_01099_b200 import _native  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def rows(pairs):
    return [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs]


def main() -> None:
    limit = 1 << 20
    want = orc.find_pairs_sorted(limit)
    ctx = _native.context(0)
    for engine in ("heavy", "screen"):
        ctx.set_engine(engine)
        got = rows(pkg.find_pairs_sorted(limit))
        assert got == want, f"{engine}: search mismatch at 2^20"
        print(f"{engine}: {len(got)} pairs below 2^20 ok", flush=True)
    ctx.set_engine("heavy")

    # a window near 2^40: the heavy classes there go through k_heavy_sieve
    lo, hi = (1 << 40) - (1 << 16), (1 << 40) + (1 << 16)
    got = pkg.search_domain(lo, hi)
    print(f"heavy window near 2^40: {len(got)} pairs, stats {pkg.last_stats()}", flush=True)

    iv = pkg.Interval(10**9, 100_001)
    ref = orc.sieve_segment(iv.start, iv.length, orc.primes_up_to(pkg.required_prime_bound(iv)))
    for ctz in (True, False):
        seg = pkg.sieve_radicals(iv, pkg.primes_up_to(pkg.required_prime_bound(iv)), ctz_fast_path=ctz)
        assert np.array_equal(seg.values, ref), f"sieve mismatch (ctz={ctz})"
    import torch

    buf = torch.empty(iv.length, dtype=torch.int64, device="cuda")
    ctx.sieve_radicals_dev(iv.start, iv.length, buf.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(buf.cpu().numpy().view(np.uint64), ref), "device sieve mismatch"
    print("exact sieve (host + device buffers) ok", flush=True)

    # build over the later half of [1, 2^17], probe with the earlier half (the reference's
    # probe takes an earlier, disjoint domain: chunked.py:344-356)
    n = 1 << 16
    vals = orc.sieve_segment(1, 2 * n + 1, orc.primes_up_to(512))
    from paper_2506_01099_b200.table import SignatureTable

    table = SignatureTable(n + 1, vals[n:-1], vals[n + 1:])
    built = table.insert_all()
    probed = table.probe_all(1, vals[:n], vals[1:n + 1])
    assert all(0 < p.m < p.n for p in built + probed)
    print(f"signature table: {len(built)} from build, {len(probed)} from probe", flush=True)
    print("sanitize workloads ok")


if __name__ == "__main__":
    main()
