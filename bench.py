#!/usr/bin/env python
"""bench.py -- integers searched per second for the Benelux-pair search on B200.

Workload (BASELINE.json configs[1]): first-kind search below S = 2^32 on one B200; with
--gpus N (torchrun, one rank per GPU) every rank owns a 2^32-integer slab of n, so the job is
the search below S = N * 2^32 (weak scaling, no data-path collective).

  value     integers searched / s with the prime tables resident in HBM: per step one
            device search (heavy generator: k_heavy_count -> cub scan -> k_heavy_screen ->
            k_heavy_exact, then k_tail -> k_tail_heavy) timed with CUDA events on the
            launching stream, L2 flushed (256 MiB write) before every step, max over ranks.
  e2e       the same metric through the public API (search_domain with a host PrimeList in
            pinned memory -> H2D copy, table build, search, D2H of the rows; for N > 1 plus
            the gather of all rows to every rank).
  roofline  the dominant stage (the candidate generator) against the HBM roofline of SURVEY.md
            section 8(d): 32 algorithmic bytes per integer searched (one 16-byte key record
            written and read), timed live with CUDA events.  The generator never touches a
            per-integer record (it visits ~0.03% of the integers), so frac >> 1 is expected;
            its own limiter, instruction issue, is reported beside it (issue_roofline, from
            the ncu launch list in profiles/); see DESIGN.md "Roofline".
  cpu_baseline  the reference's chunked Algorithm 3 (oracle/oracle.c, a C restatement of
            chunked.py:307-412 at the reference defaults: chunk 2^27, all host threads) on a
            bounded sample (one chunk build + one parallel round of probes), extrapolated to
            the full run with the reference's own schedule.

`--impl reference` prints the reference arm (rank 0 only) on the same metric and config.
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

PER_GPU = 1 << 32
BYTES_PER_INT = 32  # 16-byte record written + read
REF_CHUNK = 1 << 27  # chunked.py:24 DEFAULT_CHUNK_SIZE
REF_SUB = 1 << 24  # values of each earlier chunk one sampled probe task covers (1/8 chunk)
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


def load_traffic(engine: str) -> dict | None:
    name = "ncu_heavy_generator.json" if engine == "heavy" else "ncu_screen_traffic.json"
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


# ------------------------------------------------------------------------------------------
def reference_sample(limit: int, threads: int, rounds: int, warmup: int, log=None) -> dict:
    """The reference's chunked search (C restatement) at its defaults on a bounded sample:
    sieve+build of the last chunk once, then `warmup + rounds` parallel probe rounds of
    `threads` earlier chunks each; extrapolate the full run with the reference schedule
    (chunk i probes its i earlier chunks on `threads` workers, chunked.py:344-356)."""
    import numpy as np

    from oracle import oracle as orc

    s = REF_CHUNK
    total = orc.num_chunks(limit, s)
    last = total - 1
    need = math.isqrt(1 + total * (s - 1))
    primes = orc.primes_up_to(need)
    table = orc.ChunkTable(last, s, limit, primes)
    t_build = table.t_build
    width = min(threads, last) if last > 0 else 0
    round_times = []
    for r in range(warmup + rounds):
        lo = (r * width) % max(1, last)
        hi = min(last, lo + width)
        t_probe, _ = table.probe(lo, hi, threads, REF_SUB)
        if r >= warmup:  # scale the sampled 1/8-chunk tasks to full-chunk tasks
            round_times.append(t_probe * (width / max(1, hi - lo)) * ((s - 1) / REF_SUB))
        if log:
            log(f"reference round {r}: {hi - lo} probes in {t_probe:.2f}s")

    def full_wall(t_round: float) -> float:
        return sum(t_build + math.ceil(i / threads) * t_round for i in range(total))

    return {
        "chunk_size": s, "chunks": total, "threads": threads, "t_build_s": t_build,
        "round_s": round_times, "width": width,
        "walls_s": [full_wall(t) for t in round_times],
    }


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    limit = PER_GPU * args.gpus
    threads = os.cpu_count() or 1
    res = reference_sample(limit, threads, args.steps, args.warmup,
                           log=(lambda m: print(m, file=sys.stderr)) if args.verbose else None)
    walls = res["walls_s"]
    wall = statistics.median(walls)
    value = (limit - 1) / wall
    sample = (f"chunked.py Algorithm 3 restated in C (oracle/oracle.c) at S={limit}, chunk 2^27 "
              f"({res['chunks']} chunks), {threads} threads: chunk {res['chunks'] - 1} sieve+build "
              f"({res['t_build_s']:.1f}s) once, then per step one round of {res['width']} parallel "
              f"re-sieve+probe tasks over 2^24 of each earlier chunk's 2^27 values (x8); full-run wall "
              f"extrapolated with the reference schedule")
    line = {
        "impl": "reference",
        "metric": load_baseline_metric(),
        "value": value,
        "unit": "n/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * statistics.median(res["round_s"]),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (the integers 1..S-1; input fully determined by S)",
        "config": workload_config(args.gpus),
        "extrapolated_wall_s": wall,
        "cpu_baseline": {"value": value, "unit": "n/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "n/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def workload_config(n: int) -> dict:
    return {
        "workload": "first-kind search to S=2^32 on 1xB200 (BASELINE configs[1]); N ranks x 2^32 n each",
        "S": PER_GPU * n,
        "kinds": "first",
        "per_gpu_integers": PER_GPU,
        "parallelism": f"n-range slabs x {n}",
        "l2": "flushed before every timed step (256 MiB device write)",
    }


# ------------------------------------------------------------------------------------------
def run_ours(args) -> None:
    import numpy as np
    import torch

    world, rank, local = dist_env()
    use_dist = world > 1 or os.environ.get("BNX_FORCE_DIST") == "1"  # the latter: exercise N>1 code on one GPU
    if use_dist:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2506_01099_b200 as bp
    from paper_2506_01099_b200 import _native
    from paper_2506_01099_b200.dist import weak_shard

    def barrier():
        if use_dist:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: int) -> int:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(t)
        return int(t.item())

    lo, hi = weak_shard(PER_GPU, rank, world)
    S = PER_GPU * world
    kinds = bp.Kind.FIRST
    expected = [p for p in bp.expected_pairs_up_to(S).first_kind if lo <= p.n <= hi]
    exp_keys = [(p.m, p.n) for p in expected]

    ctx = _native.context(local)
    stream = torch.cuda.Stream(dev)  # a real stream: the library and the events share it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    # timed steps without the library's internal events: one CUDA graph per search; the
    # generator / pipeline split for the roofline comes from a separate pass with them on
    ctx.set_timing(False)

    # host prime list in pinned memory (the e2e input)
    need = math.isqrt(hi + 1)
    host_primes = bp.primes_up_to(need)
    pinned = torch.empty(len(host_primes), dtype=torch.int64, pin_memory=True)
    pinned.numpy().view(np.uint64)[:] = host_primes.primes
    plist = bp.PrimeList(pinned.numpy().view(np.uint64), host_primes.limit)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # ---- value: device-resident tables -------------------------------------------------
    ctx.prepare(hi + 1)
    for _ in range(args.warmup):
        ctx.enqueue(lo, hi, int(kinds))
        ctx.collect()
    sampler = ClockSampler(physical_gpu(local))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    screen_ms, pipe_ms, ok = [], [], True
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    wall0 = time.perf_counter()
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        ev[k][0].record(stream)
        ctx.enqueue(lo, hi, int(kinds))
        ev[k][1].record(stream)
        rows = ctx.collect()
        ok &= [(int(r["m"]), int(r["n"])) for r in rows] == exp_keys
    torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    stats = ctx.stats()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_local = sum(step_ms) / args.steps
    ms = max_over_ranks(ms_local)
    ints_local = hi - lo + 1
    ints = sum_over_ranks(ints_local)
    value = ints / (ms / 1e3)
    all_ok = bool(max_over_ranks(0.0 if ok else 1.0) == 0.0)

    if clocks["samples"] < 3:  # timed region shorter than the sampling period: sample a repeat
        sampler2 = ClockSampler(physical_gpu(local))
        sampler2.start()
        t_end = time.time() + 1.5
        while time.time() < t_end:
            ctx.enqueue(lo, hi, int(kinds))
            ctx.collect()
        c2 = sampler2.stop()
        c2["note"] = "timed region shorter than 100 ms sampling; clocks sampled over a 1.5 s repeat of the step"
        clocks = c2

    # ---- generator / pipeline split (library events between two graph launches) ----------
    ctx.set_timing(True)
    for k in range(args.warmup + max(10, args.steps // 2)):
        flush.fill_(k & 0xFF)
        ctx.enqueue(lo, hi, int(kinds))
        ctx.collect()
        if k >= args.warmup:
            s_ms, p_ms = ctx.timing()
            screen_ms.append(s_ms)
            pipe_ms.append(p_ms)
    ctx.set_timing(False)

    # ---- e2e: public API, host buffers ----------------------------------------------------
    e2e_ms = []
    d2h = 0
    for k in range(args.warmup + args.steps):
        flush.fill_(k & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record(stream)
        if use_dist:
            from paper_2506_01099_b200.dist import gather_rows

            local_rows = bp.search.search_rows(lo, hi, kinds=kinds, primes=plist, device=local)
            rows = gather_rows(local_rows)
        else:
            rows = bp.search.search_rows(lo, hi, kinds=kinds, primes=plist, device=local)
        b.record(stream)
        b.synchronize()
        if k >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
        # bnx_capi.cu read_back(): one copy of the I/O block head (counters, flags: 160 B) and PAIR_PREFIX 40-byte rows
        # (a second copy of the rows only when a search finds more than PAIR_PREFIX pairs)
        d2h = 160 + 40 * max(64, len(rows))
    e2e_ms_max = max_over_ranks(sum(e2e_ms) / len(e2e_ms))
    e2e_value = ints / (e2e_ms_max / 1e3)
    h2d = 8 * len(plist.primes)

    # ---- the same step with the byte-screen engine (visits every integer; identical rows)
    screen_engine = None
    if rank == 0 and ctx.engine() == "heavy":
        ctx.set_engine("screen")
        ctx.prepare(hi + 1)
        for _ in range(2):
            ctx.enqueue(lo, hi, int(kinds))
            ctx.collect()
        sms = []
        same = True
        for k in range(5):
            flush.fill_(k & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.enqueue(lo, hi, int(kinds))
            b.record(stream)
            rows_s = ctx.collect()
            sms.append(a.elapsed_time(b))
            same &= [(int(r["m"]), int(r["n"])) for r in rows_s] == exp_keys
        ctx.set_engine("heavy")
        screen_engine = {"engine": "screen (k_screen: one byte per integer, every integer visited)",
                         "ms_per_step": sum(sms) / len(sms), "value": ints_local / (sum(sms) / len(sms) / 1e3),
                         "unit": "n/s", "same_pairs": same}

    # ---- roofline of the dominant kernel ---------------------------------------------------
    peak, peak_src = load_peaks()
    scr_ms = sum(screen_ms) / len(screen_ms)
    achieved = BYTES_PER_INT * ints_local / (scr_ms / 1e3) / 1e9
    engine = ctx.engine()
    traffic = load_traffic(engine)
    traffic_bytes = None
    issue = None
    if traffic and traffic.get("dram_bytes_per_integer") is not None:
        traffic_bytes = traffic["dram_bytes_per_integer"] * ints_local
    if traffic and traffic.get("warp_inst_per_integer"):
        # the generator's own limiter: SM instruction issue (4 warp-instructions per SM per clock)
        props = torch.cuda.get_device_properties(dev)
        max_mhz = clocks.get("sm_max_mhz") or 1965.0
        peak_issue = props.multi_processor_count * 4 * max_mhz * 1e6
        ach_issue = traffic["warp_inst_per_integer"] * ints_local / (scr_ms / 1e3)
        issue = {"achieved": ach_issue, "peak": peak_issue, "unit": "warp-instructions/s",
                 "frac": ach_issue / peak_issue,
                 "inst_per_integer_source": f"ncu {traffic.get('source')} ({traffic['warp_inst_per_integer']:.6f} warp-inst/int)"}

    # ---- secondary: the exact radical sieve (radical.py:109-124) materialising rad(x) as
    # uint64 in HBM -- a write-bound kernel, 8 algorithmic bytes per integer
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
        sieve = {"kernel": "k_sieve_exact", "integers": n_sieve, "ms": t_ms, "achieved": gbs, "peak": peak,
                 "unit": "GB/s", "frac": gbs / peak, "bound": "hbm",
                 "bytes_per_integer": 8, "check_rad_2^30": int(out[-1].item())}
        del out
        torch.cuda.empty_cache()

    # ---- the metric's second clause: wall time to S = 2^40 (both kinds, one GPU), checked
    # against Theorem 1 (20 + 21 pairs); the device search only, tables resident
    wall40 = None
    if rank == 0 and world == 1 and not args.no_2p40:
        S40 = 1 << 40
        ctx.prepare(S40)
        ctx.enqueue(1, S40 - 1, 3)
        ctx.collect()  # warm-up
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(7)
        a_ev.record(stream)
        ctx.enqueue(1, S40 - 1, 3)
        b_ev.record(stream)
        rows40 = ctx.collect()
        exp40 = bp.expected_pairs_up_to(S40)
        want = sorted((p.m, p.n) for p in exp40.first_kind + exp40.second_kind)
        wall40 = {"S": S40, "kinds": "both", "wall_s": a_ev.elapsed_time(b_ev) / 1e3,
                  "int_per_s": (S40 - 1) / (a_ev.elapsed_time(b_ev) / 1e3), "pairs": len(rows40),
                  "matches_theorem_1": sorted((int(r["m"]), int(r["n"])) for r in rows40) == want}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        res = reference_sample(S, threads, 1, 0)
        w = res["walls_s"][0]
        cpu = {
            "value": (S - 1) / w, "unit": "n/s", "cores": threads, "kind": "port",
            "sample": (f"chunked.py Algorithm 3 restated in C (oracle/oracle.c), S=2^32, chunk 2^27, {threads} "
                       f"threads: 1 chunk sieve+build ({res['t_build_s']:.1f}s) + 1 round of {res['width']} "
                       f"parallel re-sieve+probe tasks on 2^24 of 2^27 values each (x8 = {res['round_s'][0]:.1f}s), "
                       f"extrapolated to the "
                       f"{res['chunks']}-chunk run ({w:.0f}s)"),
        }

    if rank == 0:
        line = {
            "metric": load_baseline_metric(),
            "value": value,
            "unit": "n/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": value / PAPER_INT_PER_S,
            "vs_baseline_note": "paper's own GPU code: S=2^32 (both kinds) in ~1 min (PAPER.md:255, BASELINE.md)",
            "dtype": "u64",
            "data": "synthetic (the integers 1..S-1; input fully determined by S)",
            "config": workload_config(world),
            "wall_s_to_S": ms / 1e3,
            "correct": all_ok,
            "pairs_found_rank0": len(exp_keys),
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": "n/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms_max,
                    "path": "paper_2506_01099_b200.search.search_rows(primes=PrimeList in pinned memory) -> C ABI bnx_search_domain"},
            "gpu_launches": stats["kernel_launches"] * args.steps,
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic_bytes,
                "kernel": ("heavy generator: k_heavy_count + cub scan + k_heavy_screen + k_heavy_exact"
                           if engine == "heavy" else "k_screen"),
                "engine": engine,
                "model": ("SURVEY.md 8(d): 32 B per integer (16-B record written + read); the generator keeps no "
                          "per-integer state at all, so achieved/peak > 1 measures the traffic the record design "
                          "would need and this design avoids; issue_roofline is its real limiter "
                          "(DESIGN.md 'Roofline')"),
                "peak_source": peak_src,
                "generator_ms_per_search": scr_ms,
                "pipeline_ms_per_step": sum(pipe_ms) / len(pipe_ms),
                "generator_share_of_step": scr_ms / ms_local,
                "issue_roofline": issue,
            },
            "screen_engine": screen_engine,
            "cpu_baseline": cpu,
            "sieve_roofline": sieve,
            "wall_to_2p40": wall40,
            "search_stats": stats,
            "wall_s_timed_region": wall,
        }
        print(json.dumps(line))
    if use_dist:
        torch.distributed.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
