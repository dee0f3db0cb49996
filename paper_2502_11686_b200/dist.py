"""Multi-GPU time sharding around the C ABI.

One process per GPU.  Rank r owns steps [r*M, (r+1)*M) with M = N / world a
power of two; every rank runs its local levels (ks_factor), the ranks
allgather their single boundary column (3n^2+2n+1 doubles each), and every
rank factors the P-column boundary system redundantly before its local
backward levels.  On GPUs the library does the allgather itself over its own
NCCL communicator (ks.Dist with a unique id, bench.py); the caller-driven
exchange below (torch.distributed, e.g. gloo through pinned host memory) is
what tests/test_gpu_multiproc.py and tests/test_dist_cpu.py use.  This module
holds only that host-side plumbing.
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
