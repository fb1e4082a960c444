"""Multi-GPU search: one process per GPU, no data-path exchange.

A pair (m, n) is found from its candidate n alone: every partner m of n is reached through
the residue classes of R = rad(n) rad(n+1) and verified exactly on the same rank (no other
rank's data is needed; see DESIGN.md section "Multi-GPU").  So the work splits two ways:
  * "items" (default with the device search): every rank runs the whole domain but its
    generator walks only 1/world of the (surplus class, k) items and sieve chunks
    (bnx_ctx_set_shard) -- balanced, since heavy integers thin out as n grows;
  * "slabs": contiguous slabs of n (shard_domain), as the reference's chunking would split.
The only collective is the final gather of the verified rows (a few dozen 40-byte records)
so every rank returns the same sorted list, which is independent of the number of ranks.

torch.distributed is the plumbing (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable

import numpy as np

from .signatures import BeneluxPair, pairs_from_rows

Searcher = Callable[[int, int], np.ndarray]  # (n_first, n_last) -> bnx_pair_t rows


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


def gather_rows(local: np.ndarray, group=None) -> np.ndarray:
    """All ranks' rows, concatenated in rank order (all_gather_object; tiny payload)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    bucket: list = [None] * world
    dist.all_gather_object(bucket, local.tobytes(), group=group)
    parts = [np.frombuffer(b, dtype=local.dtype) for b in bucket]
    return np.concatenate(parts) if parts else local[:0]


def find_pairs_distributed(limit: int, *, kinds=None, device: int | None = None, group=None,
                           searcher: Searcher | None = None, balance: str | None = None) -> list[BeneluxPair]:
    """Every pair m < n < limit, computed by all ranks of `group`; every rank returns the
    same list sorted by (m, n).  `balance` is "items" (default for the device search) or
    "slabs"; `searcher` overrides the device search (tests, slabs only)."""
    import torch.distributed as dist

    if limit < 3:
        raise ValueError("limit must be >= 3")
    balance = balance or ("slabs" if searcher else "items")
    if balance not in ("items", "slabs") or (balance == "items" and searcher):
        raise ValueError(f"bad balance {balance!r}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    from ._native import PAIR_DTYPE

    if balance == "items":
        from . import _native
        from .search import search_rows

        ctx = _native.context(device)
        ctx.set_shard(rank, world)
        try:
            local = search_rows(1, limit - 1, kinds=kinds, device=device)
        finally:
            ctx.set_shard(0, 1)
    else:
        run = searcher or _device_searcher(kinds, device)
        dom = shard_domain(1, limit - 1, rank, world)
        local = run(*dom) if dom else np.empty(0, PAIR_DTYPE)
    rows = gather_rows(np.ascontiguousarray(local, dtype=PAIR_DTYPE), group)
    order = np.lexsort((rows["n"], rows["m"]))
    return pairs_from_rows(rows[order])
