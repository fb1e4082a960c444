"""Per-kernel summary of one device search from an ncu launch list (run here, no GPU).

    python scripts/ncu_generator.py gpurun_out/gen.csv --integers 4294967295 \
        --out profiles/ncu_heavy_generator.json
The launch list must come from scripts/profile_search.py (two identical searches); the last
launch of every kernel is the measured search.  bench.py reads the JSON for its issue
roofline (warp instructions per integer of the candidate generator).
"""
import argparse
import csv
import json

GENERATOR = ("k_heavy_count", "DeviceScanInitKernel", "DeviceScanKernel", "k_heavy_screen", "k_heavy_sieve",
             "k_heavy_exact")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "inst": 1, "": 1}


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "")
    for g in GENERATOR + ("k_tail_heavy", "k_tail"):
        if g in base:
            return g
    return base.split("::")[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--integers", type=int, required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--source", default="")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(int(r[ii]), {"kernel": short(r[ki])})
        d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    # the second search: the launches after the last k_heavy_count's predecessor pipeline
    ids = sorted(launches)
    counts = [i for i in ids if launches[i]["kernel"] == "k_heavy_count"]
    start = counts[-1]
    last = [launches[i] for i in ids if i >= start]
    per = []
    for d in last:
        per.append({"kernel": d["kernel"], "time_ns": d.get("gpu__time_duration.sum"),
                    "warp_inst": d.get("smsp__inst_executed.sum"),
                    "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)})
    gen = [p for p in per if p["kernel"] in GENERATOR]
    tot_t = sum(p["time_ns"] for p in per)
    gen_t = sum(p["time_ns"] for p in gen)
    gen_i = sum(p["warp_inst"] for p in gen)
    gen_b = sum(p["dram_bytes"] for p in gen)
    out = {
        "integers_per_search": args.integers,
        "launches": per,
        "generator_kernels": list(GENERATOR),
        "generator_time_ns": gen_t,
        "search_time_ns": tot_t,
        "generator_share": gen_t / tot_t,
        "warp_inst_per_integer": gen_i / args.integers,
        "dram_bytes_per_integer": gen_b / args.integers,
        "dram_bytes_per_search": gen_b,
        "dominant_kernel": max(per, key=lambda p: p["time_ns"])["kernel"],
        "note": "ncu --clock-control none, serialised cold launches: shares, not absolute times",
        "source": args.source,
    }
    json.dump(out, open(args.out, "w"), indent=1)
    for p in per:
        print(f"{p['kernel']:22s} {p['time_ns'] / 1e3:9.1f} us {p['warp_inst'] / 1e6:9.2f} M warp-inst "
              f"{p['dram_bytes'] / 1e6:8.2f} MB")
    print(f"generator {gen_t / 1e3:.1f} us of {tot_t / 1e3:.1f} us; {out['warp_inst_per_integer']:.5f} warp-inst/int")


if __name__ == "__main__":
    main()
