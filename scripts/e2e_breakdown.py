"""Where the public-API time goes beyond the device search: the same search through (a) the
split-phase device path, (b) the raw C ABI bnx_search via ctypes, (c) the package API
(find_pairs -> BeneluxPair objects); CUDA events around each call, L2 flushed."""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_01099_b200 as bp  # noqa: E402
from paper_2506_01099_b200 import _native  # noqa: E402

S = 2**32
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = _native.context(0)
ctx.set_stream(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
L = _native.load()
buf = (_native.PairRow * 256)()
found = ctypes.c_size_t(0)


def timed(fn, n=60):
    ms, host = [], []
    for k in range(n):
        flush.fill_(k & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        b.record(stream)
        b.synchronize()
        if k >= 10:
            ms.append(a.elapsed_time(b))
            host.append(1e3 * (t1 - t0))
    return round(statistics.median(ms), 4), round(statistics.median(host), 4)


ctx.prepare(S)


def split():
    ctx.enqueue(1, S - 1, 1)
    ctx.collect()


print("split-phase enqueue+collect", timed(split))
print("raw ctypes bnx_search", timed(lambda: L.bnx_search(ctx.handle, S, 1, None, 0, 0, buf, 256, ctypes.byref(found))))
print("ctx.search (numpy rows)", timed(lambda: ctx.search(S, 1, None, 0)))
print("find_pairs (BeneluxPair)", timed(lambda: bp.search.find_pairs(S, kinds=1)))
rows = ctx.search(S, 1, None, 0)
t0 = time.perf_counter()
for _ in range(1000):
    bp.signatures.pairs_from_rows(rows)
print("pairs_from_rows 16 rows us", (time.perf_counter() - t0) * 1e3)
