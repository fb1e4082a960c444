"""Cold first-call phases (BNX_TRACE=1 prints them): a fresh library context per bound, CUDA
context already up.  python scripts/trace_cold.py [bounds...]"""
import os
import sys
import time

os.environ.setdefault("BNX_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

torch.zeros(1).cuda()
from paper_2506_01099_b200 import _native  # noqa: E402

bounds = [int(eval(b)) for b in sys.argv[1:]] or [2**32, 1_400_000_000_000, 2**44, 2**48]
for rep in range(2):
    for S in bounds:
        c = _native.Context(0)
        t = time.perf_counter()
        r = c.search(S, 3, None, 0)
        print(f"cold rep {rep} S={S} pairs={len(r)} {1e3 * (time.perf_counter() - t):.2f} ms", file=sys.stderr, flush=True)
        c.close()
