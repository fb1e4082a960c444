"""Summarise ncu captures for profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py --rep gpurun_out/screen.ncu-rep --launches gpurun_out/launches.csv \
        --integers 4294967295 --tag r01 --out profiles/
Writes <tag>_ncu_<kernel>.md and ncu_screen_traffic.json (DRAM bytes per integer, read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed_op_shared_atom.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        recs.append({h: (r[i], units[i]) for i, h in enumerate(head) if i < len(r)})
    return recs


def val(rec, key):
    v, u = rec[key]
    return float(v.replace(",", "")) * SCALE.get(u, 1.0), u


def launches(path: str):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        t = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        agg.setdefault(r[ki].split("(")[0].replace("void ", ""), []).append(t)
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--integers", type=int, required=True, help="integers one profiled launch screens")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--out", default="profiles")
    ap.add_argument("--peak-gbs", type=float, default=6547.5)
    ap.add_argument("--bytes-per-int", type=float, default=32.0,
                    help="algorithmic bytes per integer (32: SURVEY 8(d) record model; 8: materialised rad)")
    args = ap.parse_args()
    recs = raw(args.rep)
    rec = recs[0]
    name = rec["Kernel Name"][0] if "Kernel Name" in rec else "kernel"
    lines = [f"# ncu --set full: {name}", "", f"report: `{os.path.basename(args.rep)}` (one launch, "
             f"{args.integers} integers screened; `--clock-control none`, cold caches, serialised)", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in rec:
            lines.append(f"| {k} | {rec[k][0]} | {rec[k][1]} |")
    t, _ = val(rec, "gpu__time_duration.sum")
    rd, _ = val(rec, "dram__bytes_read.sum")
    wr, _ = val(rec, "dram__bytes_write.sum")
    insts, _ = val(rec, "smsp__inst_executed.sum")
    per_int = (rd + wr) / args.integers
    lines += ["", "Derived:", "",
              f"* duration {t * 1e3:.3f} ms -> {args.integers / t / 1e12:.3f} T integers/s under ncu",
              f"* DRAM traffic {rd + wr:.0f} B per launch = {per_int:.2e} B per integer "
              f"(SURVEY 8(d) record design: 32 B per integer)",
              f"* {insts / args.integers:.3f} warp instructions per integer "
              f"({32 * insts / args.integers:.2f} thread instructions)",
              f"* algorithmic bandwidth ({args.bytes_per_int:g} B/integer) "
              f"{args.bytes_per_int * args.integers / t / 1e9:.0f} GB/s = "
              f"{args.bytes_per_int * args.integers / t / 1e9 / args.peak_gbs:.2f} x measured HBM peak {args.peak_gbs} GB/s"]
    if args.launches:
        agg = launches(args.launches)
        total = sum(sum(v) for v in agg.values())
        lines += ["", "## Launch list (ncu --metrics gpu__time_duration.sum; shares of profiled device time)", "",
                  "| kernel | launches | avg us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) * 1e6:.1f} | {sum(v) / total:.1%} |")
    os.makedirs(args.out, exist_ok=True)
    short = "screen" if "k_screen" in name else name.split("::")[-1].split("<")[0].split("(")[0].split()[-1]
    with open(os.path.join(args.out, f"{args.tag}_ncu_{short}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if short == "screen":
        with open(os.path.join(args.out, "ncu_screen_traffic.json"), "w") as f:
            json.dump({"dram_bytes_per_integer": per_int, "dram_bytes_per_launch": rd + wr,
                       "warp_inst_per_integer": insts / args.integers,
                       "integers_per_launch": args.integers, "source": os.path.basename(args.rep),
                       "tag": args.tag}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
