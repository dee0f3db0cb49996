"""Host-side multi-GPU logic on CPU: world_size-2 gloo process groups.

The kernels need a GPU; what is covered here is the plumbing every rank runs
around them: the shard ranges (power-of-two shards, the first step of a
shard keeping its evolution row), the boundary allgather in rank order, and
the max-over-ranks timing reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_11686_b200 import dist as kdist
from paper_2502_11686_b200 import generators as gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E = 3 * 6 * 6 + 2 * 6 + 1
        send = torch.full((E * 8,), rank + 1, dtype=torch.uint8)
        send[:8] = torch.tensor([rank] * 8, dtype=torch.uint8)
        recv = torch.empty(world * E * 8, dtype=torch.uint8)
        kdist.exchange_boundary(send, recv)
        ok_gather = all(bool((recv[r * E * 8 + 8:(r + 1) * E * 8] == r + 1).all()) and
                        int(recv[r * E * 8]) == r for r in range(world))
        m = kdist.max_over_ranks(10.0 + rank)
        lo, hi = kdist.shard_range(1 << 10, rank, world)
        q.put((rank, ok_gather, m, lo, hi))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_boundary_exchange_and_timing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, ok, m, lo, hi in res:
        assert ok
        assert m == 10.0 + world - 1
        assert (lo, hi) == (rank * (1024 // world), (rank + 1) * (1024 // world))


def test_shard_range_rules():
    assert kdist.shard_range(1 << 22, 3, 8) == (3 << 19, 4 << 19)
    assert kdist.shard_range(1000, 0, 1) == (0, 1000)          # one rank: any N
    with pytest.raises(ValueError):
        kdist.shard_range(1000, 0, 8)                          # 125 not a power of two
    with pytest.raises(ValueError):
        kdist.shard_range(1 << 10, 2, 2)                       # bad rank
    with pytest.raises(ValueError):
        kdist.shard_range(3, 0, 2)


def test_shard_keeps_coupling_row():
    """A shard's first step keeps F, K, c of its (global) step: the evolution
    row to the previous shard's last state travels with the shard (no halo)."""
    p = gen.make("c2", N=64)
    lo, hi = kdist.shard_range(64, 1, 2)
    s = p.slice(lo, hi)
    np.testing.assert_array_equal(s.F[0], p.F[lo])
    np.testing.assert_array_equal(s.K[0], p.K[lo])
    np.testing.assert_array_equal(s.o, p.o[lo:hi])
    c5 = gen.make("c5", N=1 << 12)
    s5 = c5.slice(*kdist.shard_range(1 << 12, 3, 4))
    assert s5.F.shape[0] == 1 and s5.N == 1 << 10            # constant model stays stride 0
