"""Profiling aid: time k_screen at S=2^32 with parts switched off (BNX_SCREEN_SKIP bits;
results are wrong by design when bits are set).  Prints screen ms per configuration."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, torch
sys.path.insert(0, %r)
from paper_2506_01099_b200 import _native
ctx = _native.context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream); ctx.set_timing(True)
ctx.prepare(2**32)
ts = []
for k in range(13):
    ctx.enqueue(1, 2**32 - 1, 1); ctx.collect()
    if k >= 3: ts.append(ctx.timing()[0])
print(sum(ts) / len(ts))
''' % ROOT
variant = os.environ.get("BNX_SCREEN_VARIANT", "1")
for skip in [int(x) for x in os.environ.get('SKIPS', '0,1,2,4,16,3,7,15,31').split(',')]:
    env = dict(os.environ, BNX_SCREEN_SKIP=str(skip), BNX_SCREEN_VARIANT=variant)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(json.dumps({"variant": variant, "skip": skip, "screen_ms": out.stdout.strip(), "err": out.stderr[-300:] if out.returncode else ""}), flush=True)
