"""One warm-up and one measured device search of [1, S) on cuda:0 -- the command profiled by
ncu for profiles/ (the bench's step without its timing/flush scaffolding).

    ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/gen.csv \
        python scripts/profile_search.py 32
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01099_b200 import _native  # noqa: E402

e = int(sys.argv[1]) if len(sys.argv) > 1 else 32
kinds = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = _native.context(0)
if len(sys.argv) > 3:
    ctx.set_engine(sys.argv[3])
ctx.prepare(1 << e)
for _ in range(2):
    ctx.enqueue(1, (1 << e) - 1, kinds)
    rows = ctx.collect()
print(len(rows), ctx.stats())
