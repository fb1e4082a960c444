"""Where the end-to-end time of one search goes (the bench's `e2e` against its device
`value`): host wall clock of each layer of the public API, and the device time of the same
call, below one bound (default 2^32, first kind -- the bench step).

    python scripts/e2e_breakdown.py [--reps 300] [--limit 4294967296]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_01099_b200 as bp  # noqa: E402
from paper_2506_01099_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=300)
ap.add_argument("--limit", type=int, default=1 << 32)
args = ap.parse_args()
S, kinds = args.limit, int(bp.Kind.FIRST)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)  # the library and the events share it (as in bench.py)
torch.cuda.set_stream(stream)
ctx = _native.context(0)
ctx.set_stream(stream.cuda_stream)
lib = _native.load()
buf = (_native.PairRow * 4096)()
found = ctypes.c_size_t(0)
mask = bp.search.kinds_mask(kinds)


def wall(fn):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return round(statistics.median(ts), 2)


def events(fn):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return round(statistics.median(ts), 2)


def raw():
    rc = lib.bnx_search(ctx.handle, S, mask, None, 0, 0, buf, len(buf), ctypes.byref(found))
    assert rc == 0, rc


def enq_collect():
    ctx.enqueue(1, S - 1, mask)
    ctx.collect()


def device_only():
    ctx.enqueue(1, S - 1, mask)


out = {
    "limit": S,
    "wall_us": {
        "find_pairs": wall(lambda: bp.search.find_pairs(S, kinds=kinds, device=0)),
        "context.search": wall(lambda: ctx.search(S, mask, None, 0)),
        "ctypes bnx_search": wall(raw),
        "enqueue + collect": wall(enq_collect),
    },
    "event_us": {
        "find_pairs": events(lambda: bp.search.find_pairs(S, kinds=kinds, device=0)),
        "ctypes bnx_search": events(raw),
    },
}
# device time of the graph alone
ts = []
for k in range(args.reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    ctx.enqueue(1, S - 1, mask)
    b.record(stream)
    ctx.collect()
    ts.append(a.elapsed_time(b) * 1e3)
out["event_us"]["graph (enqueue only)"] = round(statistics.median(ts), 2)
t0 = time.perf_counter()
for _ in range(args.reps):
    ctx.enqueue(1, S - 1, mask)
    ctx.collect()
out["wall_us"]["enqueue + collect, mean"] = round((time.perf_counter() - t0) / args.reps * 1e6, 2)
ts = []
for _ in range(args.reps):
    t0 = time.perf_counter()
    ctx.enqueue(1, S - 1, mask)
    ts.append((time.perf_counter() - t0) * 1e6)
    ctx.collect()
out["wall_us"]["enqueue call"] = round(statistics.median(ts), 2)
print(json.dumps(out))
