"""Executed warp instructions and stall samples of one kernel grouped by source-line ranges.

    python scripts/sass_regions.py sass.csv disasm.txt k_heavy_screen bnx_heavy.cu 240-266:mask 267-290:post ...
(inputs as for scripts/sass_lines.py; lines outside every range are grouped per file)."""
import csv
import sys
from collections import defaultdict

sys.path.insert(0, __import__("os").path.dirname(__file__))
import sass_lines  # noqa: E402


def main():
    sass_csv, dis, fun, src = sys.argv[1:5]
    ranges = []
    for tok in sys.argv[5:]:
        span, name = tok.split(":", 1)
        a, b = (int(v) for v in span.split("-"))
        ranges.append((a, b, name))
    lm = sass_lines.line_map(dis, fun)
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    ai, si, ii = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [r for r in rows[2:] if len(r) > ii and r[ai].startswith("0x")]
    base = int(data[0][ai], 16)
    agg = defaultdict(lambda: [0, 0])
    for r in data:
        f, line = lm.get(int(r[ai], 16) - base, ("?", 0))
        name = f
        if f == src:
            name = next((n for a, b, n in ranges if a <= line <= b), f"{src} other")
        agg[name][0] += int(r[si] or 0)
        agg[name][1] += int(r[ii] or 0)
    ts = sum(v[0] for v in agg.values())
    ti = sum(v[1] for v in agg.values())
    for name, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:32s} inst {n / 1e6:8.2f}M {100 * n / ti:5.1f}%   stall samples {100 * s / ts:5.1f}%")


if __name__ == "__main__":
    main()
