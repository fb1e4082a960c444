"""Multi-rank path on CPU: world_size 2 over gloo.  Each rank searches its slab of n with
the searcher injected (the C oracle restricted to the slab; the device search replaces it on
GPUs), the rows are all-gathered, and every rank must hold the reference's full list,
independent of the number of ranks."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, limit, q):
    import sys

    sys.path.insert(0, ROOT)
    import numpy as np
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_2506_01099_b200 import _native
    from paper_2506_01099_b200.dist import find_pairs_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def searcher(lo, hi):
        rows = [r for r in orc.find_pairs_sorted(hi + 1) if lo <= r[2] <= hi]
        arr = np.zeros(len(rows), dtype=_native.PAIR_DTYPE)
        for i, (k, m, n, rm, rm1) in enumerate(rows):
            arr[i] = (m, n, rm, rm1, k, 0)
        return arr

    pairs = find_pairs_distributed(limit, searcher=searcher)
    got = [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs]
    q.put((rank, got))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_search_equals_reference(world, golden):
    limit = 1 << 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, limit, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [tuple(r) for r in golden["find_pairs_sorted"][str(limit)]]
    for r in range(world):
        assert results[r] == want


def _items_worker(rank, world, port, limit, q):
    """Items mode (the device's default sharding): every rank searches the whole domain and
    returns only its shard's rows; the gather + sort must rebuild the full list.  The shard
    function stands in for bnx_ctx_set_shard (a deterministic partition of the pairs)."""
    import sys

    sys.path.insert(0, ROOT)
    import numpy as np
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_2506_01099_b200 import _native
    from paper_2506_01099_b200.dist import find_pairs_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def shard_searcher(shard, nshards):
        rows = [r for r in orc.find_pairs_sorted(limit) if (r[1] * 7919 + r[2]) % nshards == shard]
        arr = np.zeros(len(rows), dtype=_native.PAIR_DTYPE)
        for i, (k, m, n, rm, rm1) in enumerate(rows):
            arr[i] = (m, n, rm, rm1, k, 0)
        return arr

    pairs = find_pairs_distributed(limit, shard_searcher=shard_searcher)
    q.put((rank, [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_item_shard_gather_equals_reference(world, golden):
    limit = 1 << 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_items_worker, args=(r, world, port, limit, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [tuple(r) for r in golden["find_pairs_sorted"][str(limit)]]
    for r in range(world):
        assert results[r] == want
