#!/usr/bin/env python
"""Time the large-n path on the paper's n = m = 500, k = 500 workload:
per-phase (eager, library events) and whole-step CUDA-graph replay.
Usage: big_time.py [N] [n]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_11686_b200 import generators as gen  # noqa: E402
from paper_2502_11686_b200 import ks, model  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].startswith("c"):   # a BASELINE config on the large-n path
    p = gen.make(sys.argv[1])
    N, n = p.N, p.n
    kw = {"big": True}
else:
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 500
    p = gen.paper_problem(N, n, seed=0)
    kw = {}
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
s = ks.Smoother(p, stream=st, **kw)
s.run(); s.check()
s.set_timing(True)
l0 = s.info()["launches"]
s.run()
tm = s.timing()
nl = s.info()["launches"] - l0
s.set_timing(False)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    s.run()
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(3):
    g.replay()
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
s.check()
sb, sf = model.step_totals(N, n, p.m_max, {"C": int(p.H.shape[0] > 1), "E": int(p.F.shape[0] > 1)})
print(json.dumps({"N": N, "n": n, "ms_per_step": ms, "steps_per_s": N / ms * 1e3, "launches": nl,
                  "phases_ms": {k: v[0] for k, v in tm.items()}, "algorithmic_flops": sf,
                  "tflops": sf / ms / 1e9, "fp64_frac": sf / ms / 1e9 / 37.0}))
