"""Per-stage device times (timing mode 2) of one item shard of the configs[3] search (first kind
below 2^40) for several shard counts, and the whole-graph time of each shard."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_01099_b200 import _native  # noqa: E402

S = 1 << 40
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = _native.context(0)
ctx.set_stream(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ctx.prepare(S)
for nsh in (1, 2, 4, 8):
    for sh in ((0,) if nsh == 1 else (0, nsh - 1)):
        ctx.set_shard(sh, nsh)
        for mode in (0, 2):
            ctx.set_timing(mode)
            ms, kt = [], []
            for k in range(8):
                flush.fill_(k)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.enqueue(1, S - 1, 1)
                b.record(stream)
                ctx.collect()
                if k >= 2:
                    ms.append(a.elapsed_time(b))
                    if mode == 2:
                        kt.append(ctx.kernel_timing())
            rec = {"nshards": nsh, "shard": sh, "timing_mode": mode, "median_ms": round(statistics.median(ms), 4)}
            if kt:
                rec["stages_ms"] = {k: round(statistics.median(d[k] for d in kt), 4) for k in kt[0]}
            print(json.dumps(rec), flush=True)
ctx.set_shard(0, 1)
ctx.set_timing(0)
