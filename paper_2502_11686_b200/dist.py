"""Multi-GPU time sharding around the C ABI.

One process per GPU.  Rank r owns steps [r*M, (r+1)*M) with M = N / world a
power of two; every rank runs its local levels (ks_factor), the ranks
allgather their single boundary column (3n^2+2n+1 doubles each) through
torch.distributed (NCCL on GPUs, gloo on CPU tests), and every rank factors
the P-column boundary system redundantly (ks_factor_boundary) before its
local backward levels.  This module holds only that host-side plumbing.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def is_pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


def shard_range(N: int, rank: int, world: int):
    """Steps [lo, hi) of `rank`; the shard size must be a power of two (the
    local levels then follow the global trailing-ones rule with no halo)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if N % world:
        raise ValueError(f"N={N} does not split over {world} ranks")
    M = N // world
    if world > 1 and (not is_pow2(M) or M < 2):
        raise ValueError(f"shard size {M} must be a power of two >= 2")
    return rank * M, (rank + 1) * M


def exchange_boundary(send: torch.Tensor, recv: torch.Tensor, group=None) -> None:
    """recv <- concat over ranks (rank order) of every rank's send buffer."""
    if recv.numel() != send.numel() * dist.get_world_size(group):
        raise ValueError("recv must hold world_size * send bytes")
    dist.all_gather_into_tensor(recv, send, group=group)


def max_over_ranks(x: float, device: Optional[torch.device] = None, group=None) -> float:
    """Max of a per-rank scalar (the timing rule: a step takes as long as the
    slowest rank)."""
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class ShardedSmoother:
    """A rank's context plus the boundary exchange: run() = whiten, local
    factor, allgather, boundary factor, solve [, selinv]."""

    def __init__(self, problem, rank: int, world: int, device="cuda", cov: bool = True, **kw):
        from . import ks
        lo, hi = shard_range(problem.N, rank, world)
        self.local = problem.slice(lo, hi) if world > 1 else problem
        self.world = world
        self.sm = ks.Smoother(self.local, device=device, cov=cov,
                              shard=(rank, world, None) if world > 1 else None, **kw)
        self.views = self.sm.boundary_tensors() if world > 1 else None

    def run(self, cov: bool = True):
        s = self.sm
        s.whiten()
        s.factor()
        if self.world > 1:
            exchange_boundary(self.views[0], self.views[1])
            s.factor_boundary()
        if cov:
            s.solve_selinv()
        else:
            s.solve()
