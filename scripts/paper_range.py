"""Reproduce the paper's bounds on one B200: every pair below 2^32, 2^40 and 1.4e12
(Theorem 1), checked against the known families.

    python scripts/paper_range.py [--bounds 2^32,2^40,1.4e12] [--kinds both]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2506_01099_b200 as bp
from oracle import theorem1  # noqa: E402


def parse_bound(s: str) -> int:
    s = s.strip()
    if s.startswith("2^"):
        return 1 << int(s[2:])
    return int(float(s))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--bounds", default="2^32,2^36,2^40,1.4e12")
    ap.add_argument("--kinds", default="both")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    results = []
    for tok in args.bounds.split(","):
        S = parse_bound(tok)
        t0 = time.perf_counter()
        pairs = bp.find_pairs(S, kinds=None if args.kinds == "both" else args.kinds)
        wall = time.perf_counter() - t0
        exp = theorem1.known_rows(S)
        got1 = sorted((p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs if p.kind == bp.Kind.FIRST)
        got2 = sorted((p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs if p.kind == bp.Kind.SECOND)
        e1 = sorted(tuple(r[1:]) for r in exp if r[0] == 1)
        e2 = sorted(tuple(r[1:]) for r in exp if r[0] == 2)
        ok = (args.kinds in ("both", "first") and got1 == e1 or args.kinds == "second") and \
             (args.kinds in ("both", "second") and got2 == e2 or args.kinds == "first")
        rec = {"S": S, "bound": tok, "wall_s": wall, "int_per_s": (S - 1) / wall, "first": len(got1),
               "second": len(got2), "matches_theorem_1": bool(ok), "stats": bp.last_stats()}
        results.append(rec)
        print(json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
