"""Per-source-line totals of an ncu SASS page: executed warp instructions and stall samples.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    cuobjdump -xelf all lib.so; nvdisasm -g bnx_heavy.sm_100a.cubin > heavy_g.txt
    python scripts/sass_lines.py sass.csv heavy_g.txt k_heavy_screen [--top 40]

The SASS page carries no line numbers; nvdisasm -g of the SAME build maps each instruction
offset to the innermost source line (inlined code is charged to its own line).
"""
import argparse
import csv
import re
from collections import defaultdict


def line_map(dis_path, fun):
    out, cur, inside = {}, None, False
    for ln in open(dis_path):
        if ln.startswith(".text.") and ln.rstrip().endswith(":"):
            inside = fun in ln
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sass_csv")
    ap.add_argument("disasm")
    ap.add_argument("fun")
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    lm = line_map(args.disasm, args.fun)
    rows = list(csv.reader(open(args.sass_csv)))
    h = rows[1]
    ai, si, ii = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [r for r in rows[2:] if len(r) > ii and r[ai].startswith("0x")]
    base = int(data[0][ai], 16)
    agg = defaultdict(lambda: [0, 0])
    tot = [0, 0]
    for r in data:
        off = int(r[ai], 16) - base
        key = lm.get(off, ("?", 0))
        s, n = int(r[si] or 0), int(r[ii] or 0)
        agg[key][0] += s
        agg[key][1] += n
        tot[0] += s
        tot[1] += n
    print(f"total samples {tot[0]}  warp instructions {tot[1]}  (mapped {len(lm)} offsets)")
    for key, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:args.top]:
        print(f"{key[0]}:{key[1]:<5} samples {s:6d} ({100 * s / max(tot[0], 1):5.1f}%)  inst {n:10d} "
              f"({100 * n / max(tot[1], 1):5.1f}%)")


if __name__ == "__main__":
    main()
