"""Profiling helper: one exact radical sieve of 2^30 integers from SIEVE_START (default 1)
into device memory (k_sieve_exact), after one warm-up call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01099_b200 import _native  # noqa: E402

ctx = _native.context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
n = 1 << 30
start = int(eval(os.environ.get("SIEVE_START", "1").replace("^", "**")))
out = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(2):
    ctx.sieve_radicals_dev(start, n, out.data_ptr())
torch.cuda.synchronize()
print(f"rad({start + n - 1}) =", int(out[-1].item()))
