"""Multi-GPU time sharding around the C ABI.

One process per GPU.  Rank r owns steps [r*M, (r+1)*M) with M = N / world a
power of two (any other N: shard_plan / pad_shard append decoupled steps up to
world*M, reading R29); every rank runs its local levels (ks_factor), the ranks
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

import numpy as np
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


def shard_plan(N: int, world: int):
    """Shard size for any N (SURVEY §8(e) "non-power-of-two chunks"):
    M = the smallest power of two >= ceil(N / world) (>= 2 for world > 1);
    rank r owns global steps [r*M, (r+1)*M) of a problem padded at its end
    to world*M steps with decoupled steps (pad_shard, reading R29).
    Returns (M, [real steps of every rank])."""
    if world < 1 or N < 1:
        raise ValueError("bad N/world")
    if world == 1:
        return N, [N]
    M = 2
    while M * world < N:
        M *= 2
    return M, [max(0, min(N, (r + 1) * M) - r * M) for r in range(world)]


def pad_shard(p, rank: int, world: int):
    """Rank `rank`'s shard of the generators.Problem `p` under shard_plan:
    its real steps [r*M, min((r+1)*M, N)) (a shard's first step keeps its
    evolution row, as Problem.slice) followed by M - real *decoupled* steps.
    A decoupled step d has F_d = 0, K_d = I, c_d = 0 and no observation
    (m_d = 0): its only row is the evolution row V_d(u_d - F_d u_{d-1} - c_d)
    = u_d, whose block on the previous state is exactly zero.
    The real steps' least-squares problem, states and covariances are
    therefore those of the unpadded problem; a decoupled step's own results
    are u_d = 0, S_dd = I.  Array plumbing only (no method arithmetic)."""
    M, real = shard_plan(p.N, world)
    lo = rank * M
    k = real[rank]
    q = p.slice(lo, lo + k) if k else p.slice(0, 1)   # all-padding rank: shapes only
    if q.nstate is not None and lo > 0 and k:
        # per-step n_i: the library cannot mask the first step's F_i (n_{i-1}
        # is on the previous rank, include/ks.h), so its ignored columns
        # >= n_{i-1} are zeroed here (the same problem)
        F = np.array(np.broadcast_to(q.F, (k,) + q.F.shape[1:]))
        F[0, :, int(p.nstate[lo - 1]):] = 0.0
        q.F = F
    if k == M:
        return q
    n, mx, pad = p.n, p.m_max, M - k

    def full(a):   # per-step copy of the k real steps (constant blocks broadcast)
        return np.broadcast_to(a, (k,) + a.shape[1:]) if a.shape[0] == 1 else a[:k]

    def cat(a, fill):
        if a is None:
            return None
        d = np.broadcast_to(np.asarray(fill, dtype=a.dtype), (pad,) + a.shape[1:])
        return np.ascontiguousarray(np.concatenate([full(a), d]))

    eye_n = np.eye(n)
    padded = type(p)(
        p.name + f"[shard {rank}/{world}, {k} + {pad} decoupled]", M, n, mx,
        np.concatenate([q.m[:k], np.zeros(pad, np.int32)]).astype(np.int32),
        cat(q.F, np.zeros((n, n))), cat(q.H, np.zeros((mx, n))), cat(q.K, eye_n),
        cat(q.L, np.eye(mx)), cat(q.o, np.zeros(mx)), cat(q.c, np.zeros(n)),
        None if q.x_true is None else np.concatenate([q.x_true[:k], np.zeros((pad, n))]),
        p.seed, dict(p.meta, shard_real=k), cat(q.Hev, eye_n),
        None if q.l is None else np.concatenate([q.l[:k], np.full(pad, n, np.int32)]),
        None if q.nstate is None else np.concatenate([q.nstate[:k], np.full(pad, n, np.int32)]))
    return padded


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
