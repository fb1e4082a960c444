#!/usr/bin/env python
"""bench.py -- integers searched per second for the Benelux-pair search on B200.

Workloads (BASELINE.json configs):
  N = 1   configs[1]: first-kind search below S = 2^32 on one B200 (the headline).
  N > 1   configs[3]: first-kind search below S = 2^40 across N GPUs (strong scaling), one
          rank per GPU (torchrun, NCCL): every rank runs the whole domain but its generator
          walks only its item shard (bnx_ctx_set_shard); the verified rows are all-gathered
          over NCCL.  Without torchrun, `--gpus N` runs the N shards one
          after another on the one visible GPU and reports the slowest (labelled "emulated").

  value     integers searched / s with the tables resident in HBM: per step one device
            search (k_heavy_count -> cub scan -> k_heavy_screen -> k_heavy_exact -> k_tail ||
            k_tail_heavy, one CUDA graph) timed with CUDA events on the launching stream, L2
            flushed (256 MiB write) before every step, max over ranks.
  e2e       the same metric through the public API (find_pairs_sorted / find_pairs_distributed:
            Python -> ctypes -> C ABI -> device -> D2H of the counters and rows; for N > 1 plus
            the NCCL gather), timed with CUDA events around the call; `e2e_cold` is the first
            call of a fresh library context (every table built on the device inside the call).
  roofline  the dominant kernel, k_heavy_screen, against its binding limit, SM instruction
            issue (4 warp-instructions per SM per clock): its warp instructions per search
            (ncu launch list, profiles/ncu_heavy_generator.json) over its live duration
            (CUDA events around the kernel, timing mode 2).  The record design of SURVEY 8(d)
            (32 B per integer through HBM) is reported as `record_design_equiv`; the HBM-bound
            kernel of the path (the exact radical sieve) as `sieve_roofline`.
  cpu_baseline / --impl reference
            the reference's chunked search (chunked.py:362-412, restated in C: oracle/oracle.c)
            run to completion at S = 2^24 (chunk 2^20, every host thread) per step -- a full,
            measured run; the quadratic 2^32 extrapolation is printed separately and labelled.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

S_HEADLINE = 1 << 32  # configs[1]
S_STRONG = 1 << 40  # configs[3]
RECORD_BYTES_PER_INT = 32  # 16-byte record written + read
REF_S, REF_CHUNK = 1 << 24, 1 << 20  # the reference arm's measured full run (2.76 s numba, 8 threads)
REF_CHUNK_2P32 = 1 << 27  # chunked.py:24 DEFAULT_CHUNK_SIZE (extrapolation only)
REF_SUB = 1 << 24
PAPER_INT_PER_S = 4294967296 / 60.0  # PAPER.md:255 "2^32 in approximately one minute"


def load_baseline_metric() -> str:
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "integers searched/sec (n/s)"


def load_peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_profile(name: str) -> dict | None:
    path = os.path.join(ROOT, "profiles", name)
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/bnx_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.out = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        self.t0 = time.time()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "note": "nvidia-smi unavailable"}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.out.close()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sms.append(float(parts[1]))
                    maxes.append(float(parts[2]))
                except ValueError:
                    continue
                for name, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        return {
            "sm_mhz": statistics.median(sms) if sms else None,
            "sm_max_mhz": max(maxes) if maxes else None,
            "reasons": sorted(reasons),
            "samples": len(sms),
        }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def physical_gpu(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if local < len(ids) and ids[local].isdigit():
            return int(ids[local])
    return local


# ---- the reference arm ------------------------------------------------------------------
def reference_full_run(threads: int) -> tuple[float, int]:
    """One complete chunked search (chunked.py:362-412, C restatement) at S = 2^24, chunk
    2^20: (wall seconds, pairs)."""
    from oracle import oracle as orc

    t0 = time.perf_counter()
    rows = orc.run_full_chunked(REF_S, REF_CHUNK, threads=threads)
    return time.perf_counter() - t0, len(rows)


def reference_extrapolation(limit: int, threads: int) -> dict:
    """EXTRAPOLATED (not measured end to end): the full chunked run to `limit` at the
    reference defaults (chunk 2^27), from one measured chunk build and one measured round of
    `threads` parallel re-sieve+probe tasks over 2^24 of each earlier chunk's values (x8),
    summed with the reference's schedule (chunk i probes its i earlier chunks in
    ceil(i / threads) rounds, chunked.py:344-356)."""
    from oracle import oracle as orc

    s = REF_CHUNK_2P32
    total = orc.num_chunks(limit, s)
    last = total - 1
    primes = orc.primes_up_to(math.isqrt(1 + total * (s - 1)))
    table = orc.ChunkTable(last, s, limit, primes)
    width = min(threads, last)
    t_probe, _ = table.probe(0, width, threads, REF_SUB)
    t_round = t_probe * ((s - 1) / REF_SUB)
    wall = sum(table.t_build + math.ceil(i / threads) * t_round for i in range(total))
    return {"S": limit, "extrapolated_wall_s": wall, "extrapolated_n_per_s": (limit - 1) / wall,
            "chunk": s, "chunks": total, "threads": threads, "measured_build_s": table.t_build,
            "measured_round_s": t_round,
            "label": "EXTRAPOLATED from one chunk build + one probe round (x8) with the reference schedule"}


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    walls = []
    pairs = 0
    for k in range(args.warmup + args.steps):
        w, pairs = reference_full_run(threads)
        if k >= args.warmup:
            walls.append(w)
        if args.verbose:
            print(f"reference step {k}: {w:.2f} s, {pairs} pairs", file=sys.stderr)
    wall = statistics.median(walls)
    value = (REF_S - 1) / wall
    sample = (f"the reference's chunked search (chunked.py:362-412) restated in C (oracle/oracle.c), run to "
              f"completion per step: S=2^24, chunk 2^20 (17 chunks, 136 chunk-pair probes), {threads} threads; "
              f"{pairs} pairs per run. A full run below 2^32 is ~100x longer per integer-range and quadratic in S, "
              f"so this per-integer rate is an upper bound for the reference at the 2^32 config")
    line = {
        "impl": "reference",
        "metric": load_baseline_metric(),
        "value": value,
        "unit": "n/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * wall,
        "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (the integers 1..S-1; input fully determined by S)",
        "config": workload_config(args.gpus),
        "measured_run": {"S": REF_S, "chunk": REF_CHUNK, "threads": threads, "wall_s_per_run": walls,
                         "pairs": pairs},
        "cpu_baseline": {"value": value, "unit": "n/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "n/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_extrapolation:
        line["extrapolated_2p32"] = reference_extrapolation(S_HEADLINE, threads)
    print(json.dumps(line), flush=True)


def workload_config(n: int) -> dict:
    if n == 1:
        return {"workload": "first-kind search to S=2^32 on 1xB200 (BASELINE configs[1])",
                "S": S_HEADLINE, "kinds": "first", "parallelism": "1 GPU",
                "l2": "flushed before every timed step (256 MiB device write)"}
    return {"workload": f"first-kind search to S=2^40 across {n}xB200 (BASELINE configs[3], strong scaling)",
            "S": S_STRONG, "kinds": "first",
            "parallelism": f"{n} item shards of the heavy generator, one rank per GPU (NCCL); rows all-gathered",
            "l2": "flushed before every timed step (256 MiB device write)"}


# ---- our arm ----------------------------------------------------------------------------
def run_ours(args) -> None:
    import numpy as np
    import torch

    world, rank, local = dist_env()
    use_dist = world > 1 or os.environ.get("BNX_FORCE_DIST") == "1"  # the latter: the N>1 code on one GPU
    emulated = world == 1 and args.gpus > 1  # N shards one after another on the one GPU
    nshards = world if world > 1 else args.gpus
    strong = nshards > 1
    if use_dist:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2506_01099_b200 as bp
    from oracle import theorem1
    from paper_2506_01099_b200 import _native

    def barrier():
        if use_dist:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    S = S_STRONG if strong else S_HEADLINE
    kinds = int(bp.Kind.FIRST)
    exp_keys = theorem1.known_pairs(S, kind=1)
    my_shards = list(range(nshards)) if emulated else [rank if world > 1 else 0]

    ctx = _native.context(local)
    stream = torch.cuda.Stream(dev)  # a real stream: the library and the events share it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_timing(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def search_shard(shard: int, k: int):
        """One timed device search of `shard` (CUDA events on the library's stream)."""
        ctx.set_shard(shard, nshards)
        flush.fill_(k & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.enqueue(1, S - 1, kinds)
        b.record(stream)
        return a, b

    # ---- value: device-resident tables -------------------------------------------------
    ctx.prepare(S)
    for k in range(args.warmup):
        for sh in my_shards:
            search_shard(sh, k)
            ctx.collect()
    sampler = ClockSampler(physical_gpu(local))
    ok = True
    step_ms = []  # per step: the slowest of this process's shards
    rows_last = {}
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    wall0 = time.perf_counter()
    for k in range(args.steps):
        per = []
        for sh in my_shards:
            a, b = search_shard(sh, k)
            rows = ctx.collect()
            per.append(a.elapsed_time(b))
            rows_last[sh] = rows
        step_ms.append(max(per))
    torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    stats = ctx.stats()
    ms_local = sum(step_ms) / len(step_ms)
    ms = max_over_ranks(ms_local)
    value = (S - 1) / (ms / 1e3)
    local_rows = np.concatenate(list(rows_last.values()))
    if use_dist and world > 1:
        from paper_2506_01099_b200.dist import gather_rows

        all_rows = gather_rows(local_rows)
    else:
        all_rows = local_rows
    ok = sorted((int(r["m"]), int(r["n"])) for r in all_rows) == exp_keys

    if clocks["samples"] < 3:  # timed region shorter than the sampling period: sample a repeat
        sampler2 = ClockSampler(physical_gpu(local))
        sampler2.start()
        t_end = time.time() + 1.5
        while time.time() < t_end:
            search_shard(my_shards[0], 0)
            ctx.collect()
        c2 = sampler2.stop()
        c2["note"] = "timed region shorter than 100 ms sampling; clocks sampled over a 1.5 s repeat of the step"
        clocks = c2

    # ---- per-kernel live times (timing mode 2: direct launches, events between kernels) ----
    ctx.set_timing(2)
    kt = []
    for k in range(args.warmup + max(10, args.steps // 2)):
        search_shard(my_shards[0], k)
        ctx.collect()
        if k >= args.warmup:
            kt.append(ctx.kernel_timing())
    ctx.set_timing(0)
    kernel_ms = {key: statistics.median(d[key] for d in kt) for key in kt[0]}

    # ---- e2e: the public API, host in / host out --------------------------------------------
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        flush.fill_(k & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record(stream)
        if world > 1:
            from paper_2506_01099_b200.dist import find_pairs_distributed

            pairs = find_pairs_distributed(S, kinds=kinds, device=local)
        elif emulated:
            pairs = bp.find_pairs_multi_gpu(S, [local] * nshards, kinds=kinds)
        else:
            pairs = bp.search.find_pairs(S, kinds=kinds, device=local)
        b.record(stream)
        b.synchronize()
        if k >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
        ok &= [(p.m, p.n) for p in pairs] == exp_keys
    e2e_ms_max = max_over_ranks(sum(e2e_ms) / len(e2e_ms))
    e2e_value = (S - 1) / (e2e_ms_max / 1e3)
    # bnx_capi.cu read_back(): one copy of the I/O block head (counters, flags: 160 B) plus
    # PAIR_PREFIX = 64 rows of 40 B; the bound and kinds travel as kernel parameters
    d2h = 160 + 40 * 64
    all_ok = bool(max_over_ranks(0.0 if ok else 1.0) == 0.0)

    # ---- e2e_cold: a fresh library context, first call (all tables built inside the call) ---
    e2e_cold = None
    if rank == 0:
        e2e_cold = {}
        for name, bound, kk in (("2^32 first kind", S_HEADLINE, 1), ("1.4e12 both kinds", theorem1.COMPLETENESS_BOUND, 3)):
            walls, ok_cold, npairs = [], True, 0
            for rep in range(2):  # rep 0 may grow the device memory pool; rep 1 reuses it
                fresh = _native.Context(local)
                try:
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    rows = fresh.search(bound, kk, None, 0)
                    walls.append(1e3 * (time.perf_counter() - t0))
                finally:
                    fresh.close()
                want = theorem1.known_pairs(bound, kind=None if kk == 3 else kk)
                ok_cold &= sorted((int(r["m"]), int(r["n"])) for r in rows) == want
                npairs = int(len(rows))
            e2e_cold[name] = {"wall_ms": walls[0], "wall_ms_second_context": walls[1],
                              "n_per_s": (bound - 1) / (walls[0] / 1e3), "pairs": npairs, "matches_theorem_1": ok_cold}
        e2e_cold["note"] = ("host wall clock around the first bnx_search of a new library context (CUDA context "
                            "already up): device prime tables, surplus-class table, graph capture, search, D2H; "
                            "the first new context may grow the device memory pool (page mapping), the second "
                            "reuses what the first freed")

    # ---- the same step with the byte-screen engine (visits every integer; identical rows)
    screen_engine = None
    if rank == 0 and not strong:
        ctx.set_engine("screen")
        ctx.prepare(S)
        for _ in range(2):
            search_shard(0, 0)
            ctx.collect()
        sms, same = [], True
        for k in range(5):
            a, b = search_shard(0, k)
            rows_s = ctx.collect()
            sms.append(a.elapsed_time(b))
            same &= sorted((int(r["m"]), int(r["n"])) for r in rows_s) == exp_keys
        ctx.set_engine("heavy")
        screen_engine = {"engine": "screen (k_screen: one byte per integer, every integer visited)",
                         "ms_per_step": sum(sms) / len(sms), "value": (S - 1) / (sum(sms) / len(sms) / 1e3),
                         "unit": "n/s", "same_pairs": same}
    ctx.set_shard(0, 1)

    # ---- roofline of the dominant kernel: k_heavy_screen, instruction issue -------------
    peak_hbm, peak_src = load_peaks()
    prof = load_profile("ncu_heavy_generator.json" if not strong else "ncu_heavy_generator_2p40.json")
    props = torch.cuda.get_device_properties(dev)
    max_mhz = clocks.get("sm_max_mhz") or 1965.0
    peak_issue = props.multi_processor_count * 4 * max_mhz * 1e6  # warp-instructions / s
    roofline = None
    if prof:
        scr = [p for p in prof["launches"] if p["kernel"] == "k_heavy_screen"]
        if scr:
            inst = scr[-1]["warp_inst"] / (nshards if strong else 1)
            t_s = kernel_ms["screen"] / 1e3
            achieved = inst / t_s
            roofline = {
                "bound": "issue", "kernel": "k_heavy_screen", "achieved": achieved, "peak": peak_issue,
                "unit": "warp-instructions/s", "frac": achieved / peak_issue,
                "traffic": scr[-1]["dram_bytes"] / (nshards if strong else 1),
                "algorithmic": {"warp_inst_per_launch": inst, "live_ms": kernel_ms["screen"],
                                "per_unit": "warp-instructions per canonical heavy integer (DESIGN.md 5)"},
                "peak_source": f"{props.multi_processor_count} SMs x 4 schedulers x {max_mhz:.0f} MHz",
                "inst_source": f"ncu {prof.get('source')}",
                "kernel_ms_live": kernel_ms,
                "screen_share_of_search": kernel_ms["screen"] / max(1e-9, sum(kernel_ms.values())),
                "record_design_equiv": {
                    "model": "SURVEY.md 8(d): 32 B per integer (16-B record written + read) -- a design this "
                             "path does not use (it visits ~0.03% of the integers); reported for comparison",
                    "achieved_gbs": RECORD_BYTES_PER_INT * (S - 1) / (ms / 1e3) / 1e9 / (nshards if strong else 1),
                    "peak_gbs": peak_hbm, "peak_source": peak_src},
            }

    # ---- secondary: the exact radical sieve (radical.py:109-124) writing rad(x) as uint64 to
    # HBM -- the path's HBM-bound kernel, 8 algorithmic bytes per integer
    sieve = None
    if rank == 0 and not args.no_sieve:
        n_sieve = 1 << 30
        out = torch.empty(n_sieve, dtype=torch.int64, device=dev)
        ctx.sieve_radicals_dev(1, n_sieve, out.data_ptr())  # warm-up: tables
        times = []
        for k in range(3):
            flush.fill_(k & 0xFF)
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            ctx.sieve_radicals_dev(1, n_sieve, out.data_ptr())
            b_ev.record(stream)
            b_ev.synchronize()
            times.append(a_ev.elapsed_time(b_ev))
        t_ms = min(times)
        gbs = 8 * n_sieve / (t_ms / 1e3) / 1e9
        check = int(out[-1].item())  # rad(2^30) = 2 (read before the fills below overwrite the buffer)
        fills = []  # the write-only ceiling of this box (the sieve only writes): fill of the same buffer
        for k in range(4):
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            out.fill_(k)
            b_ev.record(stream)
            b_ev.synchronize()
            fills.append(a_ev.elapsed_time(b_ev))
        write_peak = 8 * n_sieve / (min(fills[1:]) / 1e3) / 1e9
        # the SURVEY 8(d) sieve windows above 2^32 (u64 slots, huge progressions bucketed per
        # window), and one at 2^62
        high = {}
        for name, st in (("2^32", 1 << 32), ("2^40-2^30", (1 << 40) - n_sieve),
                         ("1.4e12-2^30", 1_400_000_000_000 - n_sieve), ("2^62", 1 << 62)):
            ctx.sieve_radicals_dev(st, n_sieve, out.data_ptr())  # warm-up: tables
            ts = []
            for k in range(3):
                flush.fill_(k & 0xFF)
                a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_ev.record(stream)
                ctx.sieve_radicals_dev(st, n_sieve, out.data_ptr())
                b_ev.record(stream)
                b_ev.synchronize()
                ts.append(a_ev.elapsed_time(b_ev))
            g = 8 * n_sieve / (min(ts) / 1e3) / 1e9
            high[name] = {"start": st, "ms": min(ts), "achieved": g, "frac": g / peak_hbm}
        sieve = {"kernel": "k_sieve_exact", "integers": n_sieve, "ms": t_ms, "achieved": gbs, "peak": peak_hbm,
                 "unit": "GB/s", "frac": gbs / peak_hbm, "bound": "hbm",
                 "bytes_per_integer": 8, "check_rad_2^30": check,
                 "slots": "32-bit shared-memory slots (window below 2^32), u64 output",
                 "write_only_peak_measured": write_peak, "frac_of_write_only_peak": gbs / write_peak,
                 "windows_above_2^32": high}
        del out
        torch.cuda.empty_cache()

    # ---- the metric's second clause: wall time to S = 2^40 (both kinds) on one GPU, and for
    # N > 1 the same-S single-GPU time of the configs[3] search (rank 0's GPU, unsharded)
    wall40 = None
    if rank == 0 and not args.no_2p40:
        wall40 = {}
        for label, kk in (("both", 3), ("first", 1)):
            if label == "first" and not strong:
                continue
            ctx.prepare(S_STRONG)
            ctx.enqueue(1, S_STRONG - 1, kk)
            ctx.collect()  # warm-up
            flush.fill_(7)
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            ctx.enqueue(1, S_STRONG - 1, kk)
            b_ev.record(stream)
            rows40 = ctx.collect()
            want = theorem1.known_pairs(S_STRONG, kind=None if kk == 3 else kk)
            wall40[label] = {"S": S_STRONG, "kinds": label, "wall_s": a_ev.elapsed_time(b_ev) / 1e3,
                             "int_per_s": (S_STRONG - 1) / (a_ev.elapsed_time(b_ev) / 1e3), "pairs": len(rows40),
                             "matches_theorem_1": sorted((int(r["m"]), int(r["n"])) for r in rows40) == want}
        if strong:
            wall40["strong_scaling_vs_1gpu"] = {
                "one_gpu_ms": 1e3 * wall40["first"]["wall_s"], "n_gpu_ms": ms,
                "speedup": 1e3 * wall40["first"]["wall_s"] / ms,
                "efficiency": 1e3 * wall40["first"]["wall_s"] / ms / nshards}

    cpu = None
    if rank == 0 and not strong and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        walls = [reference_full_run(threads)[0] for _ in range(2)]
        w = min(walls)
        cpu = {"value": (REF_S - 1) / w, "unit": "n/s", "cores": threads, "kind": "port",
               "sample": (f"the reference's chunked search (chunked.py:362-412, C restatement oracle/oracle.c) run "
                          f"to completion at S=2^24, chunk 2^20, {threads} threads: {w:.2f} s (best of 2)")}
        if not args.no_extrapolation:
            cpu["extrapolated_2p32"] = reference_extrapolation(S_HEADLINE, threads)

    if rank == 0:
        line = {
            "metric": load_baseline_metric(),
            "value": value,
            "unit": "n/s",
            "n_gpus": nshards if emulated else world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": value / PAPER_INT_PER_S,
            "vs_baseline_note": "paper's own GPU code: S=2^32 (both kinds) in ~1 min (PAPER.md:255, BASELINE.md)",
            "dtype": "u64",
            "data": "synthetic (the integers 1..S-1; input fully determined by S)",
            "config": workload_config(nshards),
            "wall_s_to_S": ms / 1e3,
            "correct": all_ok,
            "pairs": len(exp_keys),
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "n/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms_max,
                    "path": ("paper_2506_01099_b200.find_pairs_distributed -> C ABI bnx_search_domain (item shard) "
                             "-> NCCL all_gather of the rows" if world > 1 else
                             "paper_2506_01099_b200.search.find_pairs -> ctypes -> C ABI bnx_search"),
                    "h2d_note": "the search's only inputs are the bound and the kind mask (kernel parameters); "
                                "tables stay resident in the library context between calls"},
            "e2e_cold": e2e_cold,
            "gpu_launches": stats["kernel_launches"] * args.steps * len(my_shards),
            "roofline": roofline,
            "screen_engine": screen_engine,
            "cpu_baseline": cpu,
            "sieve_roofline": sieve,
            "wall_to_2p40": wall40,
            "search_stats": stats,
            "wall_s_timed_region": wall,
        }
        if emulated:
            line["emulated"] = (f"{nshards} shards run one after another on one GPU; ms_per_step is the slowest "
                                f"shard (the projected {nshards}-GPU step, no collective)")
        print(json.dumps(line), flush=True)
    if use_dist:
        torch.distributed.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extrapolation", action="store_true", help="skip the labelled 2^32 CPU extrapolation")
    ap.add_argument("--no-sieve", action="store_true", help="skip the secondary radical-sieve roofline")
    ap.add_argument("--no-2p40", action="store_true", help="skip the wall-time-to-2^40 measurement")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
