"""Write-only HBM bandwidth on this B200 (the ceiling of a kernel that only writes, like the
exact radical sieve): torch fill_ and zero_ of 8 GiB, and a read+write copy for comparison;
min of 5 with CUDA events.  One JSON line."""
import json

import torch

n = 1 << 30
a = torch.empty(n, dtype=torch.int64, device="cuda")
b = torch.empty(n, dtype=torch.int64, device="cuda")


def best(fn, bytes_moved):
    t = []
    for k in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn(k)
        e.record()
        e.synchronize()
        if k:
            t.append(s.elapsed_time(e))
    ms = min(t)
    return {"ms": ms, "GBps": bytes_moved / (ms / 1e3) / 1e9}


out = {
    "fill_int64_8GiB": best(lambda k: a.fill_(k), 8 * n),
    "zero_8GiB": best(lambda k: a.zero_(), 8 * n),
    "copy_8GiB_read_plus_write": best(lambda k: b.copy_(a), 16 * n),
}
print(json.dumps(out))
