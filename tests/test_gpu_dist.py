"""The multi-rank search with real device searches: two ranks (processes) over gloo, both on
cuda:0 (this environment has one GPU; the ranks' kernels never wait on each other, only the
final row gather is collective).  Every rank must return the reference's list for 2^24."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, limit, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2506_01099_b200.dist import find_pairs_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pairs = find_pairs_distributed(limit, device=0)
    q.put((rank, [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_device_search(world, golden):
    limit = 1 << 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, limit, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [tuple(r) for r in golden["find_pairs_sorted"][str(limit)]]
    for r in range(world):
        assert results[r] == want


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0, 0]])
def test_single_thread_multi_device_search(devices, golden):
    """bnx_search_multi (one host thread drives the GPUs): shard i on
    devices[i]; here every shard shares cuda:0.  Rows equal the single-device search and the
    reference's list, for any number of shards."""
    import paper_2506_01099_b200 as bp

    limit = 1 << 24
    got = [(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in bp.find_pairs_multi_gpu(limit, devices)]
    assert got == [tuple(r) for r in golden["find_pairs_sorted"][str(limit)]]
    big = bp.find_pairs_multi_gpu(1 << 36, devices)
    assert [(p.m, p.n, p.kind) for p in big] == [(p.m, p.n, p.kind) for p in bp.find_pairs(1 << 36)]


def _nccl_worker(port, limit, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2506_01099_b200.dist import find_pairs_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    assert dist.get_backend() == "nccl"
    pairs = find_pairs_distributed(limit, device=0)  # item shard 0 of 1; rows gathered by NCCL on cuda:0
    q.put([(int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1) for p in pairs])
    dist.destroy_process_group()


def test_nccl_row_gather_one_rank(golden):
    """The NCCL code path of dist.py (two all_gather_into_tensor calls on the rank's GPU),
    with the one rank this box has; every pair below 2^24 with its radicals."""
    limit = 1 << 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), limit, q))
    p.start()
    got = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert got == [tuple(r) for r in golden["find_pairs_sorted"][str(limit)]]
