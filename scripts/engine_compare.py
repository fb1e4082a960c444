"""Run a list of search domains on the engine selected by BNX_ENGINE (heavy | screen) and
print one JSON line per domain: pairs digest, candidate count and device timing.  Run it once
per engine and diff the outputs (the pair lists and candidate counts must agree)."""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01099_b200 import _native, search  # noqa: E402

DOMAINS = [(1, 2), (1, 100), (1, 10**4), (1, 2**20), (1, 2**24 - 1), (5_000_000, 2**24), (1, 2**28 - 1),
           (1, 2**32 - 1), (2**32, 2**33 - 1), (2**36, 2**36 + 2**32), (2**40 - 2**32, 2**40 - 1),
           (1_400_000_000_000 - 2**30, 1_400_000_000_000), (2**41 - 2**30, 2**41 - 1)]
if len(sys.argv) > 1:
    DOMAINS = [tuple(int(v) for v in d.split(":")) for d in sys.argv[1:]]

ctx = _native.context(0)
ctx.set_timing(True)
for lo, hi in DOMAINS:
    t0 = time.perf_counter()
    rows = search.search_rows(lo, hi)
    dt = time.perf_counter() - t0
    st = ctx.stats()
    tm = ctx.timing()
    key = np.ascontiguousarray(rows).tobytes()
    print(json.dumps({"engine": os.environ.get("BNX_ENGINE", "heavy"), "lo": lo, "hi": hi, "pairs": len(rows),
                      "sha": hashlib.sha256(key).hexdigest()[:16], "candidates": st["candidates"],
                      "survivors": st["survivors"], "gen_ms": tm[0], "pipeline_ms": tm[1], "wall_s": dt}), flush=True)
