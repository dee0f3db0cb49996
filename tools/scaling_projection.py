#!/usr/bin/env python
"""Projected time-sharded scaling of config 5 from single-GPU measurements
(this pool leases one GPU; NCCL refuses two ranks per GPU): for P in
1, 2, 4, 8 a rank's work is the single-GPU plan of N/P steps (bitwise the
same kernels, tests/test_gpu_parity.py::test_sharded_launch_count) plus the
boundary system.  Measured here, per P, on one B200:
  * T_local(P): CUDA-graph replay of rank P-1's whole sharded step with the
    boundary allgather replaced by the device copy of virtual shards -- i.e.
    whiten, local levels, boundary re-tiling + boundary factor tail, boundary
    backward tail, scatter, local backward levels;
the NCCL allgather of P x (3n^2+2n+1) doubles (~1 KB per rank) over
NVLink/NVSwitch is NOT measured; it is listed as an assumption (allgather_us).
Prints a table; a projection, not a multi-GPU measurement."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_11686_b200 import generators as gen  # noqa: E402
from paper_2502_11686_b200 import ks  # noqa: E402

ALLGATHER_US = float(os.environ.get("ALLGATHER_US", "15"))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
N = 1 << 22
p = gen.make("c5")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
rows = []
for P in (1, 2, 4, 8):
    M = N // P
    r = P - 1                      # the last rank (it has a left neighbour)
    q = p.slice(r * M, (r + 1) * M)
    s = ks.Smoother(q, stream=st, shard=(r, P) if P > 1 else None)
    if P > 1:
        # a plausible boundary system: every rank's send buffer after one
        # local factor (all ranks of c5 see statistically identical data)
        s.whiten(); s.factor()
        snd, rcv = s.boundary_tensors()
        rcv.copy_(snd.repeat(P))   # (values only need to be finite and full rank)

    def run():
        s.whiten()
        s.factor()
        if P > 1:
            s.factor_boundary()
        s.solve_selinv()
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    proj = ms + (ALLGATHER_US / 1e3 if P > 1 else 0.0)
    rows.append({"P": P, "local_steps": M, "rank_step_ms": ms, "projected_ms": proj,
                 "projected_steps_per_s": N / (proj / 1e3)})
    del g, s
    torch.cuda.empty_cache()
t1 = rows[0]["projected_ms"]
print(f"config 5, N = 2^22, one B200 per rank; allgather assumed {ALLGATHER_US} us (not measured)")
print("| P | steps per rank | rank step (measured, 1 GPU) ms | projected step ms | projected steps/s | projected efficiency |")
print("|---|---|---|---|---|---|")
for rw in rows:
    eff = t1 / (rw["P"] * rw["projected_ms"])
    print(f"| {rw['P']} | {rw['local_steps']} | {rw['rank_step_ms']:.3f} | {rw['projected_ms']:.3f} | "
          f"{rw['projected_steps_per_s']:.3e} | {eff:.2f} |")
print(json.dumps(rows))
