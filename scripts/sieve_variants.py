"""A/B of the exact radical sieve geometries (BNX_SIEVE_VARIANT): for each compiled variant,
in its own process, time k_sieve_exact over [1, 2^30] (min of 5, CUDA events, L2 flushed)
and hash the output plus two windows high in the range, so the variants can be compared
for speed and for identical radicals.  Prints one JSON line per variant.  [1, 2^30] runs the
32-bit-slot geometry BNX_SIEVE_NARROW (default 0; -1: the u64 variant itself); SIEVE_START
moves the timed window (e.g. 2^40, 2^62: u64 slots, huge progressions bucketed per window,
BNX_SIEVE_GBUCKETS)."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child() -> None:
    import torch

    sys.path.insert(0, ROOT)
    from paper_2506_01099_b200 import _native

    ctx = _native.context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    flush = torch.empty(1 << 26, dtype=torch.int32, device="cuda")
    n = 1 << 30
    start0 = int(eval(os.environ.get("SIEVE_START", "1").replace("^", "**")))  # timed window [start0, start0 + 2^30)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    ctx.sieve_radicals_dev(start0, n, out.data_ptr())
    times = []
    for k in range(5):
        flush.fill_(k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        ctx.sieve_radicals_dev(start0, n, out.data_ptr())
        b.record(s)
        b.synchronize()
        times.append(a.elapsed_time(b))
    h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
    hi = []
    for start in (1 << 40, 1_400_000_000_000 - (1 << 26), (1 << 48) + 12345):
        m = 1 << 26
        ctx.sieve_radicals_dev(start, m, out.data_ptr())
        torch.cuda.synchronize()
        hi.append(hashlib.sha256(out[:m].cpu().numpy().tobytes()).hexdigest()[:16])
    for start, m in ((987654321, (1 << 20) + 12345), (3, 777)):  # ragged, 8-byte aligned output
        ctx.sieve_radicals_dev(start, m, out.data_ptr() + 8)
        torch.cuda.synchronize()
        hi.append(hashlib.sha256(out[1:m + 1].cpu().numpy().tobytes()).hexdigest()[:16])
    ms = min(times)
    print(json.dumps({"variant": os.environ.get("BNX_SIEVE_VARIANT", "0"),
                      "narrow": os.environ.get("BNX_SIEVE_NARROW", "0"),
                      "start": start0, "ms": ms,
                      "GBps": 8 * n / (ms / 1e3) / 1e9, "times": times, "sha_2p30": h, "sha_high": hi}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        arg = sys.argv[1] if len(sys.argv) > 1 else "4"  # a count, or a comma-separated list
        vs = [int(v) for v in arg.split(",")] if "," in arg else list(range(int(arg))) + [0]
        for v in vs:
            env = dict(os.environ, BNX_SIEVE_VARIANT=str(v))
            r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or f'{{"variant": {v}, "error": {json.dumps(r.stderr[-400:])}}}', flush=True)
