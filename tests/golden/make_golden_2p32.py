"""Generate tests/golden/ref_pairs_2p32.json by running the UNMODIFIED reference
(`run_full_chunked(2**32, 2**28, threads=8)`, chunked.py:362-412) in this container.

Run once from the repo root (needs /root/reference and ~30 GB RAM, ~25 min):
    python tests/golden/make_golden_2p32.py
The fixture is committed; nothing at test time reads /root/reference.
"""
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import benelux_pairs as bp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

if __name__ == "__main__":
    limit, chunk = 1 << 32, 1 << 28
    threads = int(os.environ.get("THREADS", os.cpu_count() or 1))
    t0 = time.perf_counter()
    rows = [
        [int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1]
        for p in bp.run_full_chunked(limit, chunk, threads=threads)
    ]
    wall = time.perf_counter() - t0
    with open(os.path.join(HERE, "ref_pairs_2p32.json"), "w") as f:
        json.dump(
            {
                "generator": "benelux_pairs.run_full_chunked(2**32, 2**28, threads=%d)" % threads,
                "wall_s": round(wall, 1),
                "order": "chunk order, (n, m) within each chunk (chunked.py:358)",
                "rows": rows,
            },
            f,
            indent=0,
        )
    print(len(rows), "rows in", round(wall, 1), "s")
