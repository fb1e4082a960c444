"""Shard balance of one search on one GPU: runs shard i of N (bnx_ctx_set_shard) one after
another and reports each shard's device time, so the N-GPU time of bnx_search_multi /
dist.find_pairs_distributed can be bounded from one GPU (max over shards), and compares with
contiguous n-slabs.  One JSON line per (S, N, mode).

    python scripts/shard_balance.py 2^40 8
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01099_b200 import _native  # noqa: E402


def parse(v: str) -> int:
    return 2 ** int(v[2:]) if v.startswith("2^") else int(float(v))


S = parse(sys.argv[1]) if len(sys.argv) > 1 else 2**40
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = _native.context(0)
ctx.set_timing(True)
ctx.prepare(S)


def run(lo, hi):
    ctx.enqueue(lo, hi, 3)
    rows = ctx.collect()
    ctx.enqueue(lo, hi, 3)  # timed repeat (graphs captured, tables warm)
    rows = ctx.collect()
    return rows, ctx.timing()[1]


full_rows, full_ms = run(1, S - 1)
for mode in ("items", "slabs"):
    ms, npairs = [], 0
    for i in range(N):
        if mode == "items":
            ctx.set_shard(i, N)
            rows, t = run(1, S - 1)
        else:
            ctx.set_shard(0, 1)
            lo = 1 + (S - 1) * i // N
            hi = (S - 1) * (i + 1) // N
            rows, t = run(lo, hi)
        ms.append(t)
        npairs += len(rows)
    ctx.set_shard(0, 1)
    print(json.dumps({"S": S, "shards": N, "mode": mode, "one_gpu_ms": full_ms, "shard_ms": ms,
                      "max_shard_ms": max(ms), "projected_speedup": full_ms / max(ms),
                      "projected_efficiency": full_ms / max(ms) / N, "pairs": npairs,
                      "pairs_one_gpu": len(full_rows)}), flush=True)
