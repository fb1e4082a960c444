"""The reference's own numba chunked search against the C restatement (oracle/oracle.c) on
this container's cores, same S, chunk and threads (evidence that the bench's reference arm,
which runs the C port because the GPU box has no /root/reference, is representative)."""
import json, os, sys, time
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/repo")
import benelux_pairs as ref
from oracle import oracle as orc
threads = os.cpu_count()
list(ref.run_full_chunked(1000, 64, threads=threads))  # JIT warm-up
orc.run_full_chunked(1000, 64, threads=threads)
out = []
for S, s in ((1 << 20, 1 << 16), (1 << 24, 1 << 20), (1 << 26, 1 << 22)):
    t0 = time.perf_counter(); a = list(ref.run_full_chunked(S, s, threads=threads)); t_ref = time.perf_counter() - t0
    t0 = time.perf_counter(); b = orc.run_full_chunked(S, s, threads=threads); t_port = time.perf_counter() - t0
    same = [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in a] == [tuple(r) for r in b]
    rec = {"S": S, "chunk": s, "threads": threads, "reference_numba_s": t_ref, "c_port_s": t_port,
           "port_over_reference": t_port / t_ref, "same_rows": same}
    print(json.dumps(rec), flush=True); out.append(rec)
