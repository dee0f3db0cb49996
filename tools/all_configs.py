#!/usr/bin/env python
"""Step time of every BASELINE.json config (CUDA-graph replay of whiten ->
factor -> solve+SelInv, and states-only: the paper's NC variant), one GPU.
Usage: all_configs.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_11686_b200 import generators as gen  # noqa: E402
from paper_2502_11686_b200 import ks  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
out = {}
for cfg in ("c1", "c2", "c3", "c4", "c5"):
    p = gen.make(cfg)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    res = {"N": p.N, "n": p.n, "m": p.m_max}
    for variant, cov in (("states+cov", True), ("states (NC)", False)):
        s = ks.Smoother(p, stream=st, cov=cov)
        for _ in range(3):
            s.run(cov=cov)
        s.check()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            s.run(cov=cov)
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(steps):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        res[variant] = {"ms_per_step": round(ms, 4), "steps_per_s": p.N / (ms / 1e3)}
        del g, s
        torch.cuda.empty_cache()
    out[cfg] = res
    print(cfg, json.dumps(res), flush=True)
