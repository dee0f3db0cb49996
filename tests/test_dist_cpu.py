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


def test_shard_plan_any_N():
    """shard_plan: the smallest power-of-two shard covering N over the ranks;
    the real steps fill the ranks in order (padding only at the global end)."""
    assert kdist.shard_plan(1 << 22, 8) == (1 << 19, [1 << 19] * 8)
    assert kdist.shard_plan(1000, 1) == (1000, [1000])
    assert kdist.shard_plan(1000, 8) == (128, [128] * 7 + [104])
    assert kdist.shard_plan(100000, 8) == (16384, [16384] * 6 + [100000 - 6 * 16384, 0])
    assert kdist.shard_plan(20000, 8) == (4096, [4096] * 4 + [20000 - 4 * 4096, 0, 0, 0])
    assert kdist.shard_plan(3, 2) == (2, [2, 1])
    for N in range(1, 70):
        for P in (2, 3, 4, 8):
            M, real = kdist.shard_plan(N, P)
            assert M >= 2 and M & (M - 1) == 0 and M * P >= N and (M == 2 or (M // 2) * P < N)
            assert sum(real) == N and all(0 <= k <= M for k in real)


def _join(parts):
    """The global padded problem the shards describe (rank order)."""
    p0 = parts[0]

    def cat(attr):
        arrs = [getattr(q, attr) for q in parts]
        if arrs[0] is None:
            return None
        return np.concatenate([np.broadcast_to(a, (q.N,) + a.shape[1:]) for a, q in zip(arrs, parts)])
    vec = lambda attr: None if getattr(p0, attr) is None else np.concatenate([getattr(q, attr) for q in parts])
    return gen.Problem("joined", sum(q.N for q in parts), p0.n, p0.m_max,
                       np.concatenate([q.m for q in parts]), cat("F"), cat("H"), cat("K"),
                       cat("L"), cat("o"), cat("c"), None, 0, {}, cat("Hev"), vec("l"), vec("nstate"))


@pytest.mark.parametrize("cfg,N,P", [("c1", 100, 8), ("c2", 150, 3), ("c3", 77, 4), ("c5", 45, 2),
                                     ("c4", 5, 4)])
def test_padded_shards_decoupled(cfg, N, P):
    """Reading R29 pinned by the oracle: the decoupled steps pad_shard appends
    leave the real steps' states and covariances those of the unpadded problem
    (to rounding: another elimination order), and come out as u = 0, S = I."""
    import oracle
    p = gen.make(cfg, N=N)
    M, real = kdist.shard_plan(N, P)
    parts = [kdist.pad_shard(p, r, P) for r in range(P)]
    assert all(q.N == M for q in parts) and [q.meta.get("shard_real", M) for q in parts] == real
    for r, q in enumerate(parts):      # each shard's real steps are the global ones
        k = real[r]
        np.testing.assert_array_equal(q.o[:k], p.o[r * M:r * M + k])
        np.testing.assert_array_equal(q.m[:k], p.m[r * M:r * M + k])
    g = _join(parts)
    xg, Sg = oracle.smooth(g)
    xo, So = oracle.smooth(p)
    scale_x = np.abs(xo).max(1, keepdims=True)
    assert np.max(np.abs(xg[:N] - xo) / scale_x) <= 1e-10
    assert np.max(np.abs(Sg[:N] - So).reshape(N, -1).max(1) / np.abs(So).reshape(N, -1).max(1)) <= 1e-10
    assert np.array_equal(xg[N:], np.zeros_like(xg[N:]))
    np.testing.assert_allclose(Sg[N:], np.broadcast_to(np.eye(p.n), Sg[N:].shape), rtol=0, atol=1e-15)


@pytest.mark.parametrize("N,P", [(40, 2), (37, 4)])
def test_padded_shards_general_model(N, P):
    """Per-step n_i over shards: pad_shard zeroes the ignored columns
    (>= n_{i-1}) of each shard's first F_i -- the library cannot mask them
    there (include/ks.h) -- and the general-model oracle gives the unpadded
    problem's results on the joined shards (padding: u = 0, S = I)."""
    from oracle import general as og
    rng = np.random.default_rng(5 + N)
    p = gen.general_problem(rng, N, 4, m_max=4, nmin=1)
    p.F[:, :, :] += 7.0 * (np.arange(4)[None, None, :] >= np.r_[4, p.nstate[:-1]][:, None, None])  # garbage
    M, real = kdist.shard_plan(N, P)
    parts = [kdist.pad_shard(p, r, P) for r in range(P)]
    for r in range(1, P):
        if real[r]:
            assert not parts[r].F[0, :, p.nstate[r * M - 1]:].any()
    g = _join(parts)
    xg, Sg = og.smooth_general(g)
    xo, So = og.smooth_general(p)
    assert np.max(np.abs(xg[:N] - xo)) <= 1e-10 * np.abs(xo).max()
    assert np.max(np.abs(Sg[:N] - So)) <= 1e-10 * np.abs(So).max()
    assert not xg[N:].any()
