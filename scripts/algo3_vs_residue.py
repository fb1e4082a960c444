"""The paper's Algorithm 3 (chunked hash table, run on the B200) against the residue-class
search, same bound, same device.  Prints one JSON line per bound.

    python scripts/algo3_vs_residue.py [--bounds 2^24,2^28,2^32] [--chunk 2^27]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01099_b200 as bp  # noqa: E402


def parse(s):
    return 1 << int(s[2:]) if s.startswith("2^") else int(float(s))


ap = argparse.ArgumentParser()
ap.add_argument("--bounds", default="2^24,2^28,2^32")
ap.add_argument("--chunk", default="2^27")
args = ap.parse_args()
chunk = parse(args.chunk)
bp.find_pairs(1 << 20)  # warm-up
for tok in args.bounds.split(","):
    S = parse(tok)
    s = min(chunk, S)
    t0 = time.perf_counter()
    a = sorted((int(p.kind), p.m, p.n) for p in bp.run_full_chunked_table(S, s))
    t_a3 = time.perf_counter() - t0
    t0 = time.perf_counter()
    b = sorted((int(p.kind), p.m, p.n) for p in bp.find_pairs(S))
    t_rs = time.perf_counter() - t0
    print(json.dumps({"S": S, "bound": tok, "chunk": s, "chunks": bp.num_chunks(S, s), "pairs": len(a),
                      "equal": a == b, "algorithm3_s": t_a3, "residue_s": t_rs,
                      "algorithm3_int_per_s": (S - 1) / t_a3, "residue_int_per_s": (S - 1) / t_rs}), flush=True)
