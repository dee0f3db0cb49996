"""Real processes, one rank each (2 and 4), on the single leased GPU.

Each process owns its context over a power-of-two shard of the steps (other
N: the shard_plan / pad_shard decoupled padding, reading R29)
(ks_dist_create with no communicator) and runs its local levels; the
boundary exchange is the caller-driven path of include/ks.h: the rank's
`send` entry goes device -> pinned host, a world-size-2 gloo allgather,
host -> the rank's `recv` buffer, then ks_factor_boundary and the local
backward levels.  The kernels of the two processes never wait on each other
(the exchange is host-mediated), so one GPU is a faithful stand-in for two.
The gathered shards must match the oracle and, for unpadded power-of-two
shards, the single-GPU result bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, cfg, N, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from paper_2502_11686_b200 import dist as kdist
    from paper_2502_11686_b200 import generators as gen
    from paper_2502_11686_b200 import ks
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = gen.make(cfg, N=N)
        M, _ = kdist.shard_plan(N, world)     # any N: decoupled padding (R29)
        d = ks.Dist(rank, world, rank * M, world * M)
        s = ks.Smoother(kdist.pad_shard(p, rank, world), device="cuda:0", dist=d)
        s.whiten()
        s.factor()
        send, recv = s.boundary_tensors()
        send_h = send.cpu()
        recv_h = torch.empty(world * send_h.numel(), dtype=torch.uint8)
        kdist.exchange_boundary(send_h, recv_h)       # gloo, host memory
        recv.copy_(recv_h.to(recv.device))
        s.factor_boundary()
        s.solve_selinv()
        s.check()
        q.put((rank, s.states.cpu().numpy(), s.cov.cpu().numpy(), d.info()))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, None, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,N,world", [("c5", 1 << 14, 2), ("c2", 1 << 12, 2), ("c3", 1 << 11, 2),
                                         ("c5", 1 << 15, 4), ("c1", 1 << 10, 4),
                                         ("c2", 3000, 2), ("c1", 1000, 4)])
def test_processes_gloo_staged_exchange(cfg, N, world):
    import oracle
    from paper_2502_11686_b200 import generators as gen
    from paper_2502_11686_b200 import ks
    from tests.dense import rel_cov_err, rel_state_err
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, cfg, N, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
    for r, x, S, info in res:
        assert x is not None, f"rank {r}: {S}"
        assert info == {"rank": r, "nranks": world, "nccl_nranks": 0}
    x = np.concatenate([r[1] for r in res])[:N]
    S = np.concatenate([r[2] for r in res])[:N]
    p = gen.make(cfg, N=N)
    xo, So = oracle.smooth(p)
    assert rel_state_err(x, xo) <= 1e-9 and rel_cov_err(S, So) <= 1e-8
    if (N // world) & (N // world - 1) == 0 and N % world == 0:
        s1 = ks.Smoother(p)
        s1.run()
        s1.check()
        assert np.array_equal(x, s1.states.cpu().numpy()) and np.array_equal(S, s1.cov.cpu().numpy())


def test_library_nccl_communicator_one_rank():
    """ks_dist_unique_id / ks_dist_create / ks_dist_info / ks_dist_destroy on
    the hardware: libnccl is dlopen'ed, a 1-rank communicator is created by
    the library (NCCL forbids two ranks on one GPU, so this box cannot run the
    2-rank allgather; tests above cover the exchange itself), and a context
    over it runs unsharded."""
    import torch
    from paper_2502_11686_b200 import generators as gen
    from paper_2502_11686_b200 import ks
    uid = ks.Dist.unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128
    d = ks.Dist(0, 1, 0, 1000, uid=uid, device="cuda:0")
    assert d.info() == {"rank": 0, "nranks": 1, "nccl_nranks": 1}
    p = gen.make("c2", N=1000)
    s1 = ks.Smoother(p, dist=d)
    s1.run()
    s1.check()
    s2 = ks.Smoother(p)
    s2.run()
    s2.check()
    assert torch.equal(s1.states, s2.states) and torch.equal(s1.cov, s2.cov)
    del s1, d


def test_bench_multi_rank_validation_mode():
    """bench.py's multi-rank flow (shards, Dist, barriers, max over ranks, e2e,
    one JSON line from rank 0) with 2 ranks on the one leased GPU: the
    host-staged exchange stands in for NCCL, which refuses two ranks per GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--exchange", "host", "--N", str(1 << 16), "--steps", "2", "--warmup", "1",
           "--no-per-config", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "validation" in d["exchange"]
