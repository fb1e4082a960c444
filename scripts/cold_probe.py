"""Cold-call probe: a warm context searches once, then fresh library contexts make their first
search (the bench's `e2e_cold` sequence), several times over, with BNX_TRACE=1 phase times
on stderr.

    BNX_TRACE=1 python scripts/cold_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_01099_b200 import _native  # noqa: E402

torch.cuda.init()
main = _native.context(0)
main.search(1 << 32, 1, None, 0)
torch.cuda.synchronize()
out = []
for bound, kinds in ((1 << 32, 1), (1 << 32, 1), (1400000000000, 3), (1400000000000, 3), (1 << 32, 1)):
    fresh = _native.Context(0)
    try:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rows = fresh.search(bound, kinds, None, 0)
        out.append({"bound": bound, "kinds": kinds, "wall_ms": round(1e3 * (time.perf_counter() - t0), 3),
                    "pairs": int(len(rows))})
    finally:
        fresh.close()
    print(json.dumps(out[-1]), flush=True)
    print("----", file=sys.stderr, flush=True)
