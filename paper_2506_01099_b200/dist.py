"""Multi-GPU search: one process per GPU, no data-path exchange.

A pair (m, n) is found from its candidate n alone: every partner m of n is reached through
the residue classes of R = rad(n) rad(n+1) and verified exactly on the same rank (no other
rank's data is needed; see DESIGN.md section "Multi-GPU").  So the work splits two ways:
  * "items" (default with the device search): every rank runs the whole domain but its
    generator walks only 1/world of the (surplus class, k) items and sieve chunks
    (bnx_ctx_set_shard) -- balanced, since heavy integers thin out as n grows;
  * "slabs": contiguous slabs of n (shard_domain), as the reference's chunking would split.
The only collective is the final gather of the verified rows (a few dozen 40-byte records)
so every rank returns the same sorted list, which is independent of the number of ranks:
two all_gather_into_tensor calls (the row counts, then the rows padded to the largest
count), on the rank's GPU under NCCL and on the host under gloo.

torch.distributed is the plumbing (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable

import numpy as np

from .signatures import BeneluxPair, pairs_from_rows

Searcher = Callable[[int, int], np.ndarray]  # (n_first, n_last) -> bnx_pair_t rows
ShardSearcher = Callable[[int, int], np.ndarray]  # (shard, nshards) -> that item shard's rows


def shard_domain(n_first: int, n_last: int, rank: int, world: int) -> tuple[int, int] | None:
    """Contiguous slab of [n_first, n_last] owned by `rank` (None if empty).  Slabs tile the
    domain in rank order and differ in size by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    total = n_last - n_first + 1
    if total <= 0:
        return None
    base, extra = divmod(total, world)
    lo = n_first + rank * base + min(rank, extra)
    size = base + (1 if rank < extra else 0)
    return (lo, lo + size - 1) if size else None


def weak_shard(per_rank: int, rank: int, world: int) -> tuple[int, int]:
    """Weak-scaling slab: rank r owns n in [r*C + 1, (r+1)*C] (the last rank stops at
    world*C - 1, so the job is the search below S = world*C)."""
    lo = rank * per_rank + 1
    hi = (rank + 1) * per_rank
    if rank == world - 1:
        hi = world * per_rank - 1
    return lo, hi


def _device_searcher(kinds, device: int | None) -> Searcher:
    from .search import search_rows

    def run(lo: int, hi: int) -> np.ndarray:
        return search_rows(lo, hi, kinds=kinds, device=device)

    return run


def _collective_device(group):
    """Where the gather's tensors live: the current GPU under NCCL, the host otherwise."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_rows(local: np.ndarray, group=None) -> np.ndarray:
    """All ranks' rows (bnx_pair_t records), concatenated in rank order.  Two fixed-shape
    collectives: all_gather_into_tensor of the per-rank row counts, then of the rows padded
    to the largest count (5 int64 words per 40-byte row)."""
    import torch
    import torch.distributed as dist

    from ._native import PAIR_DTYPE

    local = np.ascontiguousarray(local, dtype=PAIR_DTYPE)
    world = dist.get_world_size(group)
    dev = _collective_device(group)
    counts = torch.zeros(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(counts, torch.tensor([len(local)], dtype=torch.int64, device=dev), group=group)
    counts_h = [int(c) for c in counts.cpu()]
    width = max(counts_h) if counts_h else 0
    if width == 0:
        return local[:0].copy()
    words = PAIR_DTYPE.itemsize // 8
    mine = np.zeros((width, words), dtype=np.int64)
    mine[: len(local)] = local.view(np.int64).reshape(len(local), words)
    out = torch.empty((world * width, words), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, torch.from_numpy(mine).to(dev), group=group)
    flat = out.cpu().numpy().reshape(world, width, words)
    parts = [flat[r, : counts_h[r]].copy().view(PAIR_DTYPE).reshape(-1) for r in range(world)]
    return np.concatenate(parts)


def find_pairs_distributed(limit: int, *, kinds=None, device: int | None = None, group=None,
                           primes=None, searcher: Searcher | None = None,
                           shard_searcher: ShardSearcher | None = None,
                           balance: str | None = None) -> list[BeneluxPair]:
    """Every pair m < n < limit, computed by all ranks of `group`; every rank returns the
    same list sorted by (m, n).  `balance` is "items" (default) or "slabs".  The device
    search can be replaced for tests: `shard_searcher(shard, nshards)` in items mode,
    `searcher(n_first, n_last)` in slabs mode."""
    import torch.distributed as dist

    if limit < 3:
        raise ValueError("limit must be >= 3")
    balance = balance or ("slabs" if searcher else "items")
    if balance not in ("items", "slabs") or (balance == "items" and searcher) or (
            balance == "slabs" and shard_searcher):
        raise ValueError(f"bad balance {balance!r}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    from ._native import PAIR_DTYPE

    if balance == "items" and shard_searcher is not None:
        local = shard_searcher(rank, world)
    elif balance == "items":
        from . import _native
        from .search import search_rows

        ctx = _native.context(device)
        ctx.set_shard(rank, world)
        try:
            local = search_rows(1, limit - 1, kinds=kinds, primes=primes, device=device)
        finally:
            ctx.set_shard(0, 1)
    else:
        run = searcher or _device_searcher(kinds, device)
        dom = shard_domain(1, limit - 1, rank, world)
        local = run(*dom) if dom else np.empty(0, PAIR_DTYPE)
    rows = gather_rows(np.ascontiguousarray(local, dtype=PAIR_DTYPE), group)
    order = np.lexsort((rows["n"], rows["m"]))
    return pairs_from_rows(rows[order])
