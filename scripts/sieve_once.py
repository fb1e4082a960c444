"""Profiling helper: one exact radical sieve of [1, 2^30] into device memory (k_sieve_exact)."""
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
out = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(2):
    ctx.sieve_radicals_dev(1, n, out.data_ptr())
torch.cuda.synchronize()
print("rad(2^30) =", int(out[-1].item()))
