"""Median wall of the public API call (bench's e2e step: find_pairs(2^32, first kind), CUDA
events around the call on the library's stream, L2 flushed before each call)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_01099_b200 as bp  # noqa: E402
from paper_2506_01099_b200 import _native  # noqa: E402

S = int(eval(sys.argv[1])) if len(sys.argv) > 1 else 2**32
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = _native.context(0)
ctx.set_stream(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ms = []
for k in range(60):
    flush.fill_(k & 0xFF)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    pairs = bp.search.find_pairs(S, kinds=1)
    b.record(stream)
    b.synchronize()
    if k >= 10:
        ms.append(a.elapsed_time(b))
print(os.environ.get("TAG", ""), "e2e median ms", round(statistics.median(ms), 4), "min", round(min(ms), 4), len(pairs))
