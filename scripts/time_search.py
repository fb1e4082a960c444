"""Median device time of repeated searches (the bench step: one CUDA graph, L2 flushed before
each), per domain; one JSON line per domain.  Environment switches (BNX_*) select variants.

    python scripts/time_search.py [--reps 20] [--kinds 1] [lo:hi ...]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_01099_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--kinds", type=int, default=1)
ap.add_argument("--tag", default=os.environ.get("TAG", ""))
ap.add_argument("domains", nargs="*", default=["1:4294967295", "1:1099511627775"])
args = ap.parse_args()

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = _native.context(0)
ctx.set_stream(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for d in args.domains:
    lo, hi = (int(v) for v in d.split(":"))
    ctx.prepare(hi + 1)
    for _ in range(3):
        ctx.enqueue(lo, hi, args.kinds)
        ctx.collect()
    ms = []
    for k in range(args.reps):
        flush.fill_(k & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.enqueue(lo, hi, args.kinds)
        b.record(stream)
        rows = ctx.collect()
        ms.append(a.elapsed_time(b))
    ctx.set_timing(2)
    kt = []
    for k in range(5):
        flush.fill_(k & 0xFF)
        ctx.enqueue(lo, hi, args.kinds)
        ctx.collect()
        kt.append(ctx.kernel_timing())
    ctx.set_timing(0)
    st = ctx.stats()
    print(json.dumps({"tag": args.tag, "lo": lo, "hi": hi, "pairs": len(rows), "median_ms": statistics.median(ms), "mean_ms": statistics.fmean(ms),
                      "min_ms": min(ms), "kernels_ms": {k: round(statistics.median(x[k] for x in kt), 4) for k in kt[0]},
                      "survivors": st["survivors"], "candidates": st["candidates"]}), flush=True)
